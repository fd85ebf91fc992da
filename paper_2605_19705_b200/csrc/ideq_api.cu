// Runtime and C ABI of the i-DEQ engine (include/ideq.h).
//
// The context owns: the network program (the ordered list of convolution launches
// for U_theta(z) and its input VJP), every workspace, the operator data, the solver
// state, and CUDA graphs of one iteration. All per-iteration work is enqueued on the
// caller's stream; the host only polls a 4-byte active-image counter.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/ideq.h"
#include "../../include/ideq_debug.h"
#include "common.cuh"
#include "kernels.h"

using namespace ideq;

namespace {

// ------------------------------------------------------------------ NCCL (dlopen'ed; whenever a dist descriptor is given)
typedef struct { char internal[128]; } nccl_uid;
typedef void* nccl_comm;
struct NcclApi {
  void* h = nullptr;
  int (*GetUniqueId)(nccl_uid*) = nullptr;
  int (*CommInitRank)(nccl_comm*, int, nccl_uid, int) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
  int (*CommDestroy)(nccl_comm) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  bool load(std::string& err) {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) { h = dlopen(n, RTLD_NOW | RTLD_GLOBAL); if (h) break; }
    if (!h) { err = "cannot dlopen libnccl.so.2"; return false; }
    GetUniqueId = (int (*)(nccl_uid*))dlsym(h, "ncclGetUniqueId");
    CommInitRank = (int (*)(nccl_comm*, int, nccl_uid, int))dlsym(h, "ncclCommInitRank");
    AllReduce = (int (*)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t))dlsym(h, "ncclAllReduce");
    CommDestroy = (int (*)(nccl_comm))dlsym(h, "ncclCommDestroy");
    GetErrorString = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
    if (!GetUniqueId || !CommInitRank || !AllReduce || !CommDestroy) { err = "libnccl missing symbols"; return false; }
    return true;
  }
};
NcclApi g_nccl;
constexpr int NCCL_FLOAT32 = 7, NCCL_MAX = 2;

// ------------------------------------------------------------------ program description
enum LayerKind { L_GEMM = 0, L_IMG2FEAT = 1, L_FEAT2IMG = 2, L_IMG2FEAT_TC = 4, L_RBF = 5 };

struct Layer {
  LayerKind kind;
  ConvGeom g{};
  const void* in = nullptr;   // GEMM / FEAT2IMG input (feature tensor)
  const void* wB = nullptr;   // device weights (GEMM: [kb][ncols][KC] of T; head/tail: fp32 [o][i][3][3])
  void* out = nullptr;
  const void* aux = nullptr;
  // head/tail
  const float* in_img = nullptr;
  float* out_img = nullptr;
  const float* aux_img = nullptr;
  float alpha = 0.f;
  int C = 0, wfeat = 0, epi = 0, N = 0, H = 0, W = 0;
  TcPlan* plan = nullptr;
  I2FPlan* i2f = nullptr;  // fused head (L_IMG2FEAT_TC): output tensor map
  RbfPlan* rbf = nullptr;  // fused residual block (L_RBF)
  bool tc = false;  // tcgen05 path (bf16 U-Net layers) vs FFMA path
  bool headtail = false;  // head/tail layer (profiled in the head/tail class, not the conv roofline)
  double flops = 0, bytes = 0;
  std::string name;
};

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

// In-graph timing of kernel classes (ideq_time_class): while an iteration is captured, an
// event-record node is placed wherever the kernel class of consecutive launches changes, so each
// run of same-class launches is bracketed by two events of the replayed graph.
struct SegTimer {
  cudaStream_t s = nullptr;
  int cur = -1;
  cudaEvent_t open = nullptr;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> seg[IDEQ_K_NCLASSES];
  std::vector<cudaEvent_t> all;
  cudaEvent_t rec() {
    cudaEvent_t e;
    cudaEventCreate(&e);
    all.push_back(e);
    cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
    return e;
  }
  void enter(int cls) {
    if (cls == cur) return;
    close();
    open = rec();
    cur = cls;
  }
  void close() {
    if (cur < 0) return;
    seg[cur].push_back({open, rec()});
    cur = -1;
  }
  ~SegTimer() { for (auto e : all) cudaEventDestroy(e); }
};

// The network program for one micro-batch size: forward then VJP launches, in order.
struct Program {
  std::vector<Layer> layers;
  int n_fwd = 0;
};

}  // namespace

struct ideq_ctx {
  int device = 0;
  // ideq_jfb_grad scratch, reused across calls: the tape blocks in allocation order, the split
  // partials of the weight-gradient reductions
  std::vector<std::pair<void*, size_t>> jfb_pool;
  float* jfb_ws = nullptr;
  size_t jfb_ws_n = 0;
  std::map<std::string, std::vector<uint32_t>> jfb_map;  // operand index -> blob index per layer
  std::map<std::string, TcPlan*> jfb_plans;  // 3xTF32 tcgen05 plans of the JFB passes (keyed by geometry + buffers)
  cudaStream_t stream = nullptr;
  ideq_precision prec = IDEQ_PREC_FP32;
  ideq_net_desc net{};
  std::vector<float> blob;
  int maxN = 0, H = 0, W = 0, C = 1;
  int num_sms = 148;
  std::string err;
  bool poisoned = false;
  size_t elt = 4;  // bytes per activation element

  std::vector<DevBuf> allocs;
  // weights per conv (device), keyed by name + direction
  std::map<std::string, void*> wdev;
  // feature buffers: per level 3 work buffers; saved activations
  std::vector<std::vector<void*>> lvl_buf;  // [level][3]
  std::map<std::string, void*> saved;
  // network programs keyed by micro-batch size (the full micro-batch and a smaller last one);
  // `prog` is the build target of build_program
  std::map<int, Program> progs;
  std::vector<Layer> prog;
  int n_fwd = 0;
  // workspace plan: the network's activations are allocated for `mb` images (the micro-batch);
  // the solver state (iterates, gradients, operator data) for every image of a solve
  int mb = 0;
  size_t net_bytes = 0;
  // the last solve's step arguments (class timing replays its kernels)
  bool fuse_rb = true;  // level-0 residual blocks as one launch (rbf.cu); ideq_debug_set_fusion
  bool have_last = false;
  bool last_fused = false;  // the last solve ran the whole-solve tiny-network kernel
  int last_N = 0;
  StepArgs last_a{};
  FinalizeArgs last_f{};

  // solver buffers (fp32 NCHW)
  float *X1 = nullptr, *Z = nullptr, *G = nullptr, *Hc = nullptr, *fbuf = nullptr, *fbuf2 = nullptr;
  float* partials = nullptr;
  // NEXT-1 (restart / averaging) state
  int* rk = nullptr;
  double* rsum = nullptr;
  int* flags = nullptr;
  int* nrest = nullptr;
  float* best = nullptr;
  int* k0 = nullptr;
  float* Zsum = nullptr;
  float* Xsnap = nullptr;
  int parts_cap = 0;
  int *active = nullptr, *status = nullptr, *iters = nullptr, *n_active = nullptr, *kdev = nullptr;
  int* act_list = nullptr;  // compacted active-image indices (conv tile loops of tol > 0 solves)
  float *res = nullptr, *r_now = nullptr, *rmax = nullptr, *trace = nullptr;
  int trace_cap = 65536;
  int* h_pinned = nullptr;  // host mirror of n_active
  float* dstage_y = nullptr;
  float* dstage_x = nullptr;
  size_t dstage_y_n = 0, dstage_x_n = 0;

  // operator
  bool op_set = false;
  ideq_operator_desc op{};
  int op_batch = 0;
  float* d_kern = nullptr;
  uint8_t* d_mask = nullptr;
  uint8_t* d_kmask = nullptr;  // MRI k-space mask [H][W]
  float* mhalf = nullptr;      // MRI mask on the half spectrum [H][W/2+1]
  float* d_phase = nullptr;
  // FFT operators
  float2* tw_h = nullptr;
  float2* tw_w = nullptr;
  float2* spec = nullptr;   // work spectrum
  float2* khat = nullptr;   // [H][W/2+1]
  float* dgl = nullptr;     // [H][W/2+1]

  // distribution
  int rank = 0, world = 1;
  nccl_comm comm = nullptr;

  // graphs
  cudaGraphExec_t gexec_plain = nullptr, gexec_check = nullptr;
  std::string graph_key;

  // profiling
  bool profiling = false;
  bool counting = false;  // class timing: Prof adds each launch's algorithmic work to cnt_*
  SegTimer* segt = nullptr;  // class timing: event nodes at class boundaries of the captured iteration
  double cnt_flops[IDEQ_K_NCLASSES] = {0}, cnt_bytes[IDEQ_K_NCLASSES] = {0};
  bool skip_frozen = false;  // current solve may freeze images early: kernels skip their work
  ideq_profile prof{};
  struct Ev { cudaEvent_t a, b; int cls; double flops, bytes; };
  std::vector<Ev> pending;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;

  int launches_per_iter = 0;
  bool own_stream = false;
};

namespace {

ideq_status fail(ideq_ctx* c, ideq_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) {
    c->err = buf;
    if (st == IDEQ_E_CUDA || st == IDEQ_E_NCCL) c->poisoned = true;
  }
  return st;
}

#define CK(call)                                                                                \
  do {                                                                                          \
    cudaError_t e_ = (call);                                                                    \
    if (e_ != cudaSuccess) return fail(ctx, IDEQ_E_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

ideq_status dalloc(ideq_ctx* ctx, void** p, size_t bytes) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(ctx, IDEQ_E_NOMEM, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
  }
  ctx->allocs.push_back({*p, bytes});
  return IDEQ_OK;
}

// ------------------------------------------------------------------ weights
uint16_t f2bf(float f) {  // round-to-nearest-even
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

struct WeightSlices {
  std::map<std::string, std::pair<size_t, std::vector<int>>> t;  // name -> offset, shape
};

bool slice_weights(const ideq_net_desc& n, WeightSlices& ws, size_t& total) {
  size_t o = 0;
  auto add = [&](const std::string& name, std::vector<int> shp) {
    size_t k = 1;
    for (int s : shp) k *= (size_t)s;
    ws.t[name] = {o, shp};
    o += k;
  };
  const int C = n.channels;
  if (n.arch == IDEQ_NET_TINY3) {
    const int w = n.widths[0];
    add("c1", {w, C, 3, 3});
    add("c2", {w, w, 3, 3});
    add("c3", {C, w, 3, 3});
  } else {
    const int* w = n.widths;
    add("head", {w[0], C, 3, 3});
    for (int l = 0; l < 4; ++l) {
      for (int r = 0; r < n.res_blocks; ++r) {
        add("e" + std::to_string(l) + "." + std::to_string(r) + ".A", {w[l], w[l], 3, 3});
        add("e" + std::to_string(l) + "." + std::to_string(r) + ".B", {w[l], w[l], 3, 3});
      }
      if (l < 3) add("down" + std::to_string(l), {w[l + 1], w[l], 2, 2});
    }
    for (int l = 2; l >= 0; --l) {
      add("up" + std::to_string(l), {w[l + 1], w[l], 2, 2});
      for (int r = 0; r < n.res_blocks; ++r) {
        add("d" + std::to_string(l) + "." + std::to_string(r) + ".A", {w[l], w[l], 3, 3});
        add("d" + std::to_string(l) + "." + std::to_string(r) + ".B", {w[l], w[l], 3, 3});
      }
    }
    add("tail", {C, w[0], 3, 3});
  }
  total = o;
  return true;
}

// Build the [kb][ncols][KC] GEMM operand for one conv direction (host fp32).
//   kind 0: conv3x3 fwd, 1: conv3x3 adjoint, 2: down fwd, 3: down adjoint, 4: up fwd, 5: up adjoint.
std::vector<float> gemm_weights(int kind, const float* Wt, const std::vector<int>& shp, int KC, int& ncols,
                                int& ntaps, int& ktap) {
  std::vector<float> B;
  if (kind == 0 || kind == 1) {  // W [co][ci][3][3]
    const int co_n = shp[0], ci_n = shp[1];
    ncols = kind == 0 ? co_n : ci_n;
    ktap = kind == 0 ? ci_n : co_n;
    ntaps = 9;
    const int nch = ktap / KC;
    B.assign((size_t)9 * nch * ncols * KC, 0.f);
    for (int t = 0; t < 9; ++t) {
      const int a = t / 3, b = t % 3;
      for (int ch = 0; ch < nch; ++ch)
        for (int n = 0; n < ncols; ++n)
          for (int k = 0; k < KC; ++k) {
            const int kk = ch * KC + k;
            const int co = kind == 0 ? n : kk, ci = kind == 0 ? kk : n;
            B[(((size_t)(t * nch + ch)) * ncols + n) * KC + k] = Wt[(((size_t)co * ci_n + ci) * 3 + a) * 3 + b];
          }
    }
  } else if (kind == 2 || kind == 5) {  // patch GEMM on the fine grid: taps a, K = (b, c)
    // down: Wd [co][ci][2][2], out cols co, k = (b, ci)       -> Wd[co][ci][a][b]
    // upT : Wu [ci][co][2][2], out cols ci(coarse), k=(b, co) -> Wu[ci][co][a][b]
    const int o_n = shp[0], f_n = shp[1];  // down: o=co(coarse) f=ci(fine); up: o=ci(coarse) f=co(fine)
    ncols = o_n;
    ktap = 2 * f_n;
    ntaps = 2;
    const int nch = ktap / KC;
    B.assign((size_t)2 * nch * ncols * KC, 0.f);
    for (int a = 0; a < 2; ++a)
      for (int ch = 0; ch < nch; ++ch)
        for (int n = 0; n < ncols; ++n)
          for (int k = 0; k < KC; ++k) {
            const int kk = ch * KC + k;
            const int b = kk / f_n, f = kk % f_n;
            B[(((size_t)(a * nch + ch)) * ncols + n) * KC + k] = Wt[(((size_t)n * f_n + f) * 2 + a) * 2 + b];
          }
  } else if (kind == 6) {  // im2col'd 3x3 head: W [o][c][3][3], k = c*9 + a*3 + b < 9c, K = 32
    const int o_n = shp[0], c_n = shp[1];
    ncols = o_n;
    ktap = 32;
    ntaps = 1;
    B.assign((size_t)ncols * KC, 0.f);
    for (int n = 0; n < ncols; ++n)
      for (int k = 0; k < 9 * c_n && k < 32; ++k) B[(size_t)n * KC + k] = Wt[(size_t)n * c_n * 9 + k];
  } else {  // 3: down adjoint, 4: up fwd -- 1x1 on the coarse grid, cols = (a, b, fine channel)
    // downT: Wd [co][ci][2][2], input coarse g (co), cols (a,b,ci): Wd[k][ci][a][b]
    // up   : Wu [ci][co][2][2], input coarse x (ci), cols (a,b,co): Wu[k][co][a][b]
    const int k_n = shp[0], f_n = shp[1];
    ncols = 4 * f_n;
    ktap = k_n;
    ntaps = 1;
    const int nch = ktap / KC;
    B.assign((size_t)nch * ncols * KC, 0.f);
    for (int ch = 0; ch < nch; ++ch)
      for (int n = 0; n < ncols; ++n)
        for (int k = 0; k < KC; ++k) {
          const int kk = ch * KC + k;
          const int a = n / (2 * f_n), b = (n / f_n) % 2, f = n % f_n;
          B[(((size_t)ch) * ncols + n) * KC + k] = Wt[(((size_t)kk * f_n + f) * 2 + a) * 2 + b];
        }
  }
  return B;
}

// 3x3 weights of the adjoint of a head/tail conv: W~[i][o][a][b] = W[o][i][2-a][2-b].
std::vector<float> flip_transpose3x3(const float* Wt, int o_n, int i_n) {
  std::vector<float> F((size_t)i_n * o_n * 9);
  for (int o = 0; o < o_n; ++o)
    for (int i = 0; i < i_n; ++i)
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
          F[(((size_t)i * o_n + o) * 3 + a) * 3 + b] = Wt[(((size_t)o * i_n + i) * 3 + (2 - a)) * 3 + (2 - b)];
  return F;
}

// K-block width: the bf16 tcgen05 path stages 32/64 channels (64B/128B swizzle rows), the 3xTF32
// path 32 fp32 channels (128B rows); the FFMA path walks 16 channels at a time.
int pick_kc(bool tc, bool x3, int ktap) {
  if (tc) return x3 ? 32 : ((ktap % 64 == 0) ? 64 : 32);
  return 16;
}
int pick_kc(bool tc, int ktap) { return pick_kc(tc, false, ktap); }

// The U-Net's convolutions run on tcgen05 in both precisions: bf16 operands (headline) or fp32
// operands as 3xTF32 (the parity mode, every width a multiple of 32). The C <-> w0 head / tail
// run on tcgen05 in bf16 and on the FFMA path in fp32; the tiny C1 net is FFMA.
bool use_tc(ideq_ctx* ctx) {
  if (ctx->net.arch != IDEQ_NET_UNET4) return false;
  if (ctx->prec == IDEQ_PREC_BF16) return true;
  for (int l = 0; l < 4; ++l)
    if (ctx->net.widths[l] % 32) return false;
  return true;
}
bool use_x3(ideq_ctx* ctx) { return ctx->prec == IDEQ_PREC_FP32 && use_tc(ctx); }
bool use_tc_headtail(ideq_ctx* ctx) { return ctx->prec == IDEQ_PREC_BF16 && use_tc(ctx); }

// 3xTF32 operand split on the host: hi = w rounded to tf32 (round to nearest, ties away from zero,
// as cvt.rna.tf32.f32), lo = (w - hi) rounded the same way (|w - hi - lo| <= 2^-22 |w|).
float tf32_rna(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

ideq_status upload_gemm_weights(ideq_ctx* ctx, const std::string& key, const std::vector<float>& B) {
  void* d = nullptr;
  const size_t n = B.size();
  ideq_status st = dalloc(ctx, &d, n * ctx->elt);
  if (st) return st;
  if (ctx->prec == IDEQ_PREC_BF16) {
    std::vector<uint16_t> hb(n);
    for (size_t i = 0; i < n; ++i) hb[i] = f2bf(B[i]);
    CK(cudaMemcpy(d, hb.data(), n * 2, cudaMemcpyHostToDevice));
  } else {
    CK(cudaMemcpy(d, B.data(), n * 4, cudaMemcpyHostToDevice));
  }
  ctx->wdev[key] = d;
  return IDEQ_OK;
}

ideq_status upload_f32(ideq_ctx* ctx, const std::string& key, const std::vector<float>& v) {
  void* d = nullptr;
  ideq_status st = dalloc(ctx, &d, v.size() * 4);
  if (st) return st;
  CK(cudaMemcpy(d, v.data(), v.size() * 4, cudaMemcpyHostToDevice));
  ctx->wdev[key] = d;
  return IDEQ_OK;
}

// ------------------------------------------------------------------ geometry builders
void tile_grid(ConvGeom& g) {
  g.Wt = g.OW < 128 ? g.OW : 128;
  g.R = 128 / g.Wt;
  if (g.R > g.OH) g.R = g.OH;
  if (g.R < 1) g.R = 1;
  g.tiles_h = (g.OH + g.R - 1) / g.R;
  g.tiles_w = (g.OW + g.Wt - 1) / g.Wt;
}

// kind as in gemm_weights. Hin/Win: spatial size of the tensor the layer READS.
ConvGeom make_geom(int kind, int N, int Hin, int Win, int cin_tensor, int ncols, int KC, int ktap, int epi) {
  ConvGeom g{};
  g.N = N;
  g.KC = KC;
  g.nchunk = ktap / KC;
  g.epi = epi;
  g.ncols = ncols;
  if (kind == 0 || kind == 1) {
    g.inC = cin_tensor; g.inW = Win; g.inP = 1; g.inH = Hin;
    g.OH = Hin; g.OW = Win;
    g.ntaps = 9;
    for (int t = 0; t < 9; ++t) {
      const int a = t / 3, b = t % 3;
      g.dh[t] = kind == 0 ? a - 1 : 1 - a;
      g.dw[t] = kind == 0 ? b - 1 : 1 - b;
      g.dp[t] = 0;
    }
    g.OHo = Hin; g.OWo = Win; g.osh = 1; g.osw = 1; g.OCp = ncols; g.CB = ncols;
  } else if (kind == 2 || kind == 5) {  // fine input -> coarse output
    g.inC = 2 * cin_tensor; g.inW = Win / 2; g.inP = 2; g.inH = Hin / 2;
    g.OH = Hin / 2; g.OW = Win / 2;
    g.ntaps = 2;
    for (int t = 0; t < 2; ++t) { g.dh[t] = 0; g.dw[t] = 0; g.dp[t] = t; }
    g.OHo = Hin / 2; g.OWo = Win / 2; g.osh = 1; g.osw = 1; g.OCp = ncols; g.CB = ncols;
  } else if (kind == 6) {  // plain 1x1 on the im2col buffer
    g.inC = cin_tensor; g.inW = Win; g.inP = 1; g.inH = Hin;
    g.OH = Hin; g.OW = Win;
    g.ntaps = 1;
    g.dh[0] = 0; g.dw[0] = 0; g.dp[0] = 0;
    g.OHo = Hin; g.OWo = Win; g.osh = 1; g.osw = 1; g.OCp = ncols; g.CB = ncols;
  } else {  // coarse input -> fine output (scatter)
    g.inC = cin_tensor; g.inW = Win; g.inP = 1; g.inH = Hin;
    g.OH = Hin; g.OW = Win;
    g.ntaps = 1;
    g.dh[0] = 0; g.dw[0] = 0; g.dp[0] = 0;
    const int fine_c = ncols / 4;
    g.OHo = 2 * Hin; g.osh = 2; g.CB = 2 * fine_c; g.OWo = Win; g.osw = 1; g.OCp = 2 * fine_c;
  }
  tile_grid(g);
  return g;
}

int act_epi(ideq_ctx* ctx, int epi) {
  if (ctx->net.act == IDEQ_ACT_IDENTITY && (epi == EPI_SOFTPLUS || epi == EPI_SIGMUL)) return EPI_STORE;
  return epi;
}

// Core of every implicit-GEMM layer: `Wt` is the conv tensor of shape `shp` in the blob layout
// of its kind (kind 6 = the im2col'd head, shape [w][C][3][3]); `key` names the uploaded
// GEMM operand so each (conv, direction) is re-arranged and uploaded once.
ideq_status add_gemm_w(ideq_ctx* ctx, const std::string& key, const float* Wt, const std::vector<int>& shp, int kind,
                       int N, int Hin, int Win, const void* in, void* out, const void* aux, int epi,
                       const std::string& lname, Layer** out_layer = nullptr) {
  Layer L;
  L.kind = L_GEMM;
  L.name = lname;
  int ncols = 0, ntaps = 0, ktap = 0;
  // shape-derived quantities; cin_tensor = channel count of the READ tensor
  if (kind == 0) { ncols = shp[0]; ktap = shp[1]; }
  else if (kind == 1) { ncols = shp[1]; ktap = shp[0]; }
  else if (kind == 2 || kind == 5) { ncols = shp[0]; ktap = 2 * shp[1]; }
  else if (kind == 6) { ncols = shp[0]; ktap = 32; }
  else { ncols = 4 * shp[1]; ktap = shp[0]; }
  const int cin_tensor = (kind == 2 || kind == 5) ? ktap / 2 : ktap;
  L.tc = use_tc(ctx);
  const bool x3 = L.tc && ctx->prec == IDEQ_PREC_FP32;
  const int KC = kind == 6 ? 32 : pick_kc(L.tc, x3, ktap);
  if (!ctx->wdev.count(key)) {
    std::vector<float> B = gemm_weights(kind, Wt, shp, KC, ncols, ntaps, ktap);
    if (x3) {  // tf32 hi / lo halves
      std::vector<float> lo(B.size());
      for (size_t i = 0; i < B.size(); ++i) {
        const float h = tf32_rna(B[i]);
        lo[i] = tf32_rna(B[i] - h);
        B[i] = h;
      }
      ideq_status st = upload_gemm_weights(ctx, key + "#lo", lo);
      if (st) return st;
    }
    ideq_status st = upload_gemm_weights(ctx, key, B);
    if (st) return st;
  }
  L.g = make_geom(kind, N, Hin, Win, cin_tensor, ncols, KC, ktap, epi == EPI_IMG ? EPI_IMG : act_epi(ctx, epi));
  L.in = in;
  L.wB = ctx->wdev[key];
  L.out = out;
  L.aux = aux;
  const double P = (double)N * L.g.OH * L.g.OW;
  L.flops = 2.0 * P * ncols * (double)(L.g.ntaps * ktap);
  const double in_elems = (double)N * L.g.inH * L.g.inW * L.g.inP * L.g.inC;
  const double out_elems = P * ncols;
  L.bytes = ctx->elt * (in_elems + out_elems * ((L.g.epi == EPI_RESADD || L.g.epi == EPI_SIGMUL) ? 2.0 : 1.0)) +
            ctx->elt * (double)ncols * L.g.ntaps * ktap;
  if (L.tc) {
    if (!tc_supported(L.g, x3)) return fail(ctx, IDEQ_E_UNSUPPORTED, "layer %s: geometry not supported by tcgen05 path", lname.c_str());
    char err[256] = {0};
    L.plan = tc_make_plan(L.g, x3, in, L.wB, x3 ? ctx->wdev[key + "#lo"] : nullptr, out, aux, ctx->num_sms, err,
                          sizeof(err));
    if (!L.plan) return fail(ctx, IDEQ_E_CUDA, "layer %s: %s", lname.c_str(), err);
    tc_plan_set_active(L.plan, ctx->act_list, ctx->n_active);  // frozen images cost nothing
  }
  ctx->prog.push_back(L);
  if (out_layer) *out_layer = &ctx->prog.back();
  return IDEQ_OK;
}

ideq_status add_gemm(ideq_ctx* ctx, const std::string& wname, int kind, int N, int Hin, int Win, const void* in,
                     void* out, const void* aux, int epi, const std::string& lname) {
  WeightSlices ws;
  size_t tot;
  slice_weights(ctx->net, ws, tot);
  auto& sl = ws.t[wname];
  const std::string key = wname + "#" + std::to_string(kind) + (use_tc(ctx) ? "tc" : "simt");
  return add_gemm_w(ctx, key, ctx->blob.data() + sl.first, sl.second, kind, N, Hin, Win, in, out, aux, epi, lname);
}

// Tensor-core head/tail (bf16 U-Net). Image -> features (head, tail adjoint): one fused kernel
// builds the K = 32 im2col row of each pixel in shared memory and runs a 1x1 tcgen05 GEMM.
// Features -> image (tail, head adjoint): a 3x3 tcgen05 conv with the C output columns padded
// to 16 (zero weights) and the EPI_IMG epilogue writing fp32 NCHW planes (+ alpha * aux).
ideq_status add_tc_img2feat(ideq_ctx* ctx, const std::string& wname, bool adjoint, int N, const float* in_img,
                            void* out_feat, const std::string& lname) {
  WeightSlices ws;
  size_t tot;
  slice_weights(ctx->net, ws, tot);
  auto& sl = ws.t[wname];
  const float* Wt = ctx->blob.data() + sl.first;
  const int o_n = sl.second[0], i_n = sl.second[1];
  std::vector<float> w;                 // [w0][C][3][3]
  if (adjoint) w = flip_transpose3x3(Wt, o_n, i_n);   // tail [C][w0] -> [w0][C]
  else w.assign(Wt, Wt + (size_t)o_n * i_n * 9);
  const int wo = adjoint ? i_n : o_n, ci = adjoint ? o_n : i_n;
  // fused im2col + 1x1 tcgen05 GEMM (one kernel); the weights are the K = 32 GEMM operand
  const std::string key = wname + (adjoint ? "#i2cT" : "#i2c") + "tc";
  if (!ctx->wdev.count(key)) {
    int ncols = 0, ntaps = 0, ktap = 0;
    std::vector<float> B = gemm_weights(6, w.data(), {wo, ci, 3, 3}, 32, ncols, ntaps, ktap);
    ideq_status st = upload_gemm_weights(ctx, key, B);
    if (st) return st;
  }
  if (wo != 32 && wo != 64) return fail(ctx, IDEQ_E_UNSUPPORTED, "head width %d: fused head needs 32 or 64", wo);
  Layer L;
  L.kind = L_IMG2FEAT_TC;
  L.name = lname;
  L.in_img = in_img;
  L.wB = ctx->wdev[key];
  L.out = out_feat;
  L.N = N; L.C = ctx->C; L.H = ctx->H; L.W = ctx->W;
  L.wfeat = wo;
  L.headtail = true;
  {
    char err[256] = {0};
    L.i2f = img2feat_make_plan((__nv_bfloat16*)out_feat, N, ctx->H, ctx->W, wo, err, sizeof(err));
    if (!L.i2f) return fail(ctx, IDEQ_E_CUDA, "layer %s: %s", lname.c_str(), err);
  }
  L.flops = 2.0 * N * ctx->H * ctx->W * 9.0 * ci * wo;
  L.bytes = (double)N * ctx->H * ctx->W * (4.0 * ctx->C + 2.0 * wo);
  ctx->prog.push_back(L);
  return IDEQ_OK;
}

ideq_status add_tc_feat2img(ideq_ctx* ctx, const std::string& wname, bool adjoint, int N, const void* in_feat,
                            float* out_img, const float* aux_img, float alpha, const std::string& lname) {
  WeightSlices ws;
  size_t tot;
  slice_weights(ctx->net, ws, tot);
  auto& sl = ws.t[wname];
  const float* Wt = ctx->blob.data() + sl.first;
  const int o_n = sl.second[0], i_n = sl.second[1];
  std::vector<float> wp;
  std::vector<int> shp;
  int kind;
  // the C <= 3 image columns padded to an MMA N of 16 (zero weights): the layer is bound by the
  // shared-memory operand reads, which N = 16 cuts from 5 KB to 4.5 KB per MMA
  constexpr int NP = 16;
  if (!adjoint) {  // tail [C][w0][3][3] -> [16][w0][3][3], rows >= C zero
    wp.assign((size_t)NP * i_n * 9, 0.f);
    std::copy(Wt, Wt + (size_t)o_n * i_n * 9, wp.begin());
    shp = {NP, i_n, 3, 3};
    kind = 0;
  } else {         // head [w0][C][3][3] -> [w0][16][3][3], columns >= C zero; kind 1 = adjoint
    wp.assign((size_t)o_n * NP * 9, 0.f);
    for (int o = 0; o < o_n; ++o)
      for (int i = 0; i < i_n; ++i)
        for (int t = 0; t < 9; ++t) wp[((size_t)o * NP + i) * 9 + t] = Wt[((size_t)o * i_n + i) * 9 + t];
    shp = {o_n, NP, 3, 3};
    kind = 1;
  }
  Layer* L = nullptr;
  ideq_status st = add_gemm_w(ctx, wname + (adjoint ? "#imgT" : "#img"), wp.data(), shp, kind, N, ctx->H, ctx->W,
                              in_feat, nullptr, nullptr, EPI_IMG, lname, &L);
  if (st) return st;
  L->headtail = true;
  L->out_img = out_img;
  L->aux_img = aux_img;
  L->alpha = alpha;
  L->flops = 2.0 * N * ctx->H * ctx->W * 9.0 * ctx->C * (adjoint ? o_n : i_n);
  tc_plan_set_image(L->plan, out_img, aux_img, alpha, ctx->C);
  return IDEQ_OK;
}

ideq_status add_headtail(ideq_ctx* ctx, LayerKind kind, const std::string& wname, bool adjoint, int N,
                         const float* in_img, const void* in_feat, void* out_feat, float* out_img, const void* aux,
                         const float* aux_img, float alpha, int epi, const std::string& lname) {
  WeightSlices ws;
  size_t tot;
  slice_weights(ctx->net, ws, tot);
  auto& sl = ws.t[wname];
  const float* Wt = ctx->blob.data() + sl.first;
  const int o_n = sl.second[0], i_n = sl.second[1];
  const std::string key = wname + (adjoint ? "#T" : "#F");
  if (!ctx->wdev.count(key)) {
    std::vector<float> v;
    if (adjoint) v = flip_transpose3x3(Wt, o_n, i_n);
    else v.assign(Wt, Wt + (size_t)o_n * i_n * 9);
    ideq_status st = upload_f32(ctx, key, v);
    if (st) return st;
  }
  Layer L;
  L.kind = kind;
  L.name = lname;
  L.wB = ctx->wdev[key];
  L.N = N; L.H = ctx->H; L.W = ctx->W;
  L.C = ctx->C;
  // feature width: image->feature layers produce it, feature->image layers consume it
  if (kind == L_IMG2FEAT) L.wfeat = adjoint ? i_n : o_n;
  else L.wfeat = adjoint ? o_n : i_n;
  L.in_img = in_img;
  L.in = in_feat;
  L.out = out_feat;
  L.out_img = out_img;
  L.aux = aux;
  L.aux_img = aux_img;
  L.alpha = alpha;
  L.epi = act_epi(ctx, epi);
  const double P = (double)N * ctx->H * ctx->W;
  L.flops = 2.0 * P * 9.0 * o_n * i_n;
  L.bytes = P * (4.0 * ctx->C + ctx->elt * L.wfeat * ((aux || aux_img) ? 2.0 : 1.0));
  ctx->prog.push_back(L);
  return IDEQ_OK;
}

// Fused residual block at level 0 (rbf.cu): the two 3x3 convolutions of one block in one launch.
// Forward: x = t, out = t', act = the saved activation a (written). VJP: x = g, out = g', act = a
// (read). The GEMM operands are those of the two unfused layers (kind 0 forward, kind 1 adjoint).
bool use_rbf(ideq_ctx* ctx, int l) {
  return ctx->prec == IDEQ_PREC_BF16 && ctx->net.arch == IDEQ_NET_UNET4 && l == 0 && ctx->net.act == IDEQ_ACT_SOFTPLUS &&
         rbf_supported(ctx->W, ctx->net.widths[0]) && ctx->fuse_rb;
}

ideq_status add_rbf(ideq_ctx* ctx, bool vjp, const std::string& nA, const std::string& nB, int N, int H, int W,
                    const void* x, void* out, void* act, const std::string& lname) {
  WeightSlices ws;
  size_t tot;
  slice_weights(ctx->net, ws, tot);
  const int kind = vjp ? 1 : 0;
  const std::string n1 = vjp ? nB : nA, n2 = vjp ? nA : nB;  // VJP: B^T first, then A^T
  const void* w[2];
  for (int i = 0; i < 2; ++i) {
    const std::string& nm = i == 0 ? n1 : n2;
    const std::string key = nm + "#" + std::to_string(kind) + "tc";
    if (!ctx->wdev.count(key)) {
      int ncols = 0, ntaps = 0, ktap = 0;
      auto& sl = ws.t[nm];
      std::vector<float> B = gemm_weights(kind, ctx->blob.data() + sl.first, sl.second, 32, ncols, ntaps, ktap);
      ideq_status st = upload_gemm_weights(ctx, key, B);
      if (st) return st;
    }
    w[i] = ctx->wdev[key];
  }
  const int C = ctx->net.widths[0];
  ConvGeom g = make_geom(kind, N, H, W, C, C, 32, C, EPI_STORE);
  Layer L;
  L.kind = L_RBF;
  L.name = lname;
  L.tc = true;
  L.in = x;
  L.out = out;
  L.aux = act;
  L.flops = 2.0 * (2.0 * N * H * W * 9.0 * C * C);
  L.bytes = 3.0 * (double)N * H * W * C * ctx->elt;  // read x (+ a), write a (forward) and the output
  char err[256] = {0};
  L.rbf = rbf_make_plan(vjp, N, H, W, g.dh, g.dw, g.dh, g.dw, (const __nv_bfloat16*)w[0], (const __nv_bfloat16*)w[1],
                        x, out, act, ctx->num_sms, err, sizeof(err));
  if (!L.rbf) return fail(ctx, IDEQ_E_CUDA, "layer %s: %s", lname.c_str(), err);
  rbf_set_active(L.rbf, ctx->act_list, ctx->n_active);
  ctx->prog.push_back(L);
  return IDEQ_OK;
}

std::string rb(const char* p, int l, int r, const char* ab) {
  return std::string(p) + std::to_string(l) + "." + std::to_string(r) + "." + ab;
}

// Build the forward + VJP program for batch N (buffers sized for maxN at create).
ideq_status build_program_impl(ideq_ctx* ctx, int N);
ideq_status build_program(ideq_ctx* ctx, int N) {
  if (ctx->progs.count(N)) return IDEQ_OK;
  ctx->prog.clear();
  ideq_status st = build_program_impl(ctx, N);
  if (st) {
    for (auto& L : ctx->prog) { if (L.plan) tc_free_plan(L.plan); if (L.i2f) img2feat_free_plan(L.i2f); if (L.rbf) rbf_free_plan(L.rbf); }
    ctx->prog.clear();
    return st;
  }
  Program& P = ctx->progs[N];
  P.layers.swap(ctx->prog);
  P.n_fwd = ctx->n_fwd;
  ctx->graph_key.clear();
  return IDEQ_OK;
}

ideq_status build_program_impl(ideq_ctx* ctx, int N) {
  const auto& n = ctx->net;
  const int C = ctx->C;
  ideq_status st;
  if (n.arch == IDEQ_NET_TINY3) {
    void* a1 = ctx->saved["a1"];
    void* a2 = ctx->saved["a2"];
    void* q = ctx->lvl_buf[0][0];
    void* q1 = ctx->lvl_buf[0][1];
    const int H = ctx->H, W = ctx->W;
    if ((st = add_headtail(ctx, L_IMG2FEAT, "c1", false, N, ctx->Z, nullptr, a1, nullptr, nullptr, nullptr, 0.f,
                           EPI_SOFTPLUS, "c1")))
      return st;
    if ((st = add_gemm(ctx, "c2", 0, N, H, W, a1, a2, nullptr, EPI_SOFTPLUS, "c2"))) return st;
    if ((st = add_headtail(ctx, L_FEAT2IMG, "c3", false, N, nullptr, a2, nullptr, ctx->Hc, nullptr,
                           n.identity_skip ? nullptr : ctx->Z, n.identity_skip ? 0.f : -1.f, EPI_STORE, "c3")))
      return st;
    ctx->n_fwd = (int)ctx->prog.size();
    if ((st = add_headtail(ctx, L_IMG2FEAT, "c3", true, N, ctx->Hc, nullptr, q, nullptr, a2, nullptr, 0.f,
                           EPI_SIGMUL, "c3T")))
      return st;
    if ((st = add_gemm(ctx, "c2", 1, N, H, W, q, q1, a1, EPI_SIGMUL, "c2T"))) return st;
    if ((st = add_headtail(ctx, L_FEAT2IMG, "c1", true, N, nullptr, q1, nullptr, ctx->G, nullptr,
                           n.identity_skip ? nullptr : ctx->Hc, n.identity_skip ? 0.f : -1.f, EPI_STORE, "c1T")))
      return st;
  } else {
    const int R = n.res_blocks;
    int Hl[4], Wl[4];
    for (int l = 0; l < 4; ++l) { Hl[l] = ctx->H >> l; Wl[l] = ctx->W >> l; }
    auto B = [&](int l, int i) { return ctx->lvl_buf[l][i]; };
    const bool tc = use_tc_headtail(ctx);
    const float* skip_aux_z = n.identity_skip ? nullptr : ctx->Z;
    const float* skip_aux_c = n.identity_skip ? nullptr : ctx->Hc;
    const float skip_alpha = n.identity_skip ? 0.f : -1.f;
    // ---- forward
    st = tc ? add_tc_img2feat(ctx, "head", false, N, ctx->Z, B(0, 0), "head")
            : add_headtail(ctx, L_IMG2FEAT, "head", false, N, ctx->Z, nullptr, B(0, 0), nullptr, nullptr, nullptr, 0.f,
                           EPI_STORE, "head");
    if (st) return st;
    int cur[4] = {0, 0, 0, 0};
    int skip_idx[3] = {0, 0, 0};
    for (int l = 0; l < 4; ++l) {
      for (int r = 0; r < R; ++r) {
        void* a = ctx->saved["e" + std::to_string(l) + "." + std::to_string(r)];
        const int o = cur[l] == 0 ? 1 : 0;
        if (use_rbf(ctx, l)) {
          if ((st = add_rbf(ctx, false, rb("e", l, r, "A"), rb("e", l, r, "B"), N, Hl[l], Wl[l], B(l, cur[l]), B(l, o), a,
                            rb("e", l, r, "AB"))))
            return st;
        } else {
          if ((st = add_gemm(ctx, rb("e", l, r, "A"), 0, N, Hl[l], Wl[l], B(l, cur[l]), a, nullptr, EPI_SOFTPLUS,
                             rb("e", l, r, "A"))))
            return st;
          if ((st = add_gemm(ctx, rb("e", l, r, "B"), 0, N, Hl[l], Wl[l], a, B(l, o), B(l, cur[l]), EPI_RESADD,
                             rb("e", l, r, "B"))))
            return st;
        }
        cur[l] = o;
      }
      if (l < 3) {
        skip_idx[l] = cur[l];
        if ((st = add_gemm(ctx, "down" + std::to_string(l), 2, N, Hl[l], Wl[l], B(l, cur[l]), B(l + 1, 0), nullptr,
                           EPI_STORE, "down" + std::to_string(l))))
          return st;
        cur[l + 1] = 0;
      }
    }
    for (int l = 2; l >= 0; --l) {
      const int o = skip_idx[l] == 0 ? 1 : 0;
      if ((st = add_gemm(ctx, "up" + std::to_string(l), 4, N, Hl[l + 1], Wl[l + 1], B(l + 1, cur[l + 1]), B(l, o),
                         B(l, skip_idx[l]), EPI_RESADD, "up" + std::to_string(l))))
        return st;
      cur[l] = o;
      for (int r = 0; r < R; ++r) {
        void* a = ctx->saved["d" + std::to_string(l) + "." + std::to_string(r)];
        const int o2 = cur[l] == 0 ? 1 : 0;
        if (use_rbf(ctx, l)) {
          if ((st = add_rbf(ctx, false, rb("d", l, r, "A"), rb("d", l, r, "B"), N, Hl[l], Wl[l], B(l, cur[l]), B(l, o2),
                            a, rb("d", l, r, "AB"))))
            return st;
        } else {
          if ((st = add_gemm(ctx, rb("d", l, r, "A"), 0, N, Hl[l], Wl[l], B(l, cur[l]), a, nullptr, EPI_SOFTPLUS,
                             rb("d", l, r, "A"))))
            return st;
          if ((st = add_gemm(ctx, rb("d", l, r, "B"), 0, N, Hl[l], Wl[l], a, B(l, o2), B(l, cur[l]), EPI_RESADD,
                             rb("d", l, r, "B"))))
            return st;
        }
        cur[l] = o2;
      }
    }
    st = tc ? add_tc_feat2img(ctx, "tail", false, N, B(0, cur[0]), ctx->Hc, skip_aux_z, skip_alpha, "tail")
            : add_headtail(ctx, L_FEAT2IMG, "tail", false, N, nullptr, B(0, cur[0]), nullptr, ctx->Hc, nullptr,
                           skip_aux_z, skip_alpha, EPI_STORE, "tail");
    if (st) return st;
    ctx->n_fwd = (int)ctx->prog.size();
    // ---- VJP, cotangent Hc
    st = tc ? add_tc_img2feat(ctx, "tail", true, N, ctx->Hc, B(0, 0), "tailT")
            : add_headtail(ctx, L_IMG2FEAT, "tail", true, N, ctx->Hc, nullptr, B(0, 0), nullptr, nullptr, nullptr, 0.f,
                           EPI_STORE, "tailT");
    if (st) return st;
    int g[4] = {0, 0, 0, 0};
    int gs[3] = {0, 0, 0};
    auto rb_vjp = [&](const char* p, int l, int r) -> ideq_status {
      void* a = ctx->saved[std::string(p) + std::to_string(l) + "." + std::to_string(r)];
      const int o = g[l] == 0 ? 1 : 0;
      ideq_status s2;
      // q = (B^T g) . sp'(a) ; g' = g + A^T q
      if (use_rbf(ctx, l)) {
        if ((s2 = add_rbf(ctx, true, rb(p, l, r, "A"), rb(p, l, r, "B"), N, Hl[l], Wl[l], B(l, g[l]), B(l, o), a,
                          rb(p, l, r, "BTAT"))))
          return s2;
        g[l] = o;
        return IDEQ_OK;
      }
      if ((s2 = add_gemm(ctx, rb(p, l, r, "B"), 1, N, Hl[l], Wl[l], B(l, g[l]), B(l, 2), a, EPI_SIGMUL,
                         rb(p, l, r, "BT"))))
        return s2;
      if ((s2 = add_gemm(ctx, rb(p, l, r, "A"), 1, N, Hl[l], Wl[l], B(l, 2), B(l, o), B(l, g[l]), EPI_RESADD,
                         rb(p, l, r, "AT"))))
        return s2;
      g[l] = o;
      return IDEQ_OK;
    };
    for (int l = 0; l <= 2; ++l) {
      for (int r = R - 1; r >= 0; --r)
        if ((st = rb_vjp("d", l, r))) return st;
      gs[l] = g[l];
      if ((st = add_gemm(ctx, "up" + std::to_string(l), 5, N, Hl[l], Wl[l], B(l, g[l]), B(l + 1, 0), nullptr,
                         EPI_STORE, "up" + std::to_string(l) + "T")))
        return st;
      g[l + 1] = 0;
    }
    for (int l = 3; l >= 0; --l) {
      if (l < 3) {
        const int o = gs[l] == 0 ? 1 : 0;
        if ((st = add_gemm(ctx, "down" + std::to_string(l), 3, N, Hl[l + 1], Wl[l + 1], B(l + 1, g[l + 1]), B(l, o),
                           B(l, gs[l]), EPI_RESADD, "down" + std::to_string(l) + "T")))
          return st;
        g[l] = o;
      }
      for (int r = R - 1; r >= 0; --r)
        if ((st = rb_vjp("e", l, r))) return st;
    }
    st = tc ? add_tc_feat2img(ctx, "head", true, N, B(0, g[0]), ctx->G, skip_aux_c, skip_alpha, "headT")
            : add_headtail(ctx, L_FEAT2IMG, "head", true, N, nullptr, B(0, g[0]), nullptr, ctx->G, nullptr, skip_aux_c,
                           skip_alpha, EPI_STORE, "headT");
    if (st) return st;
  }
  return IDEQ_OK;
}

// ------------------------------------------------------------------ launching (optionally profiled)
cudaEvent_t next_event(ideq_ctx* ctx) {
  if (ctx->ev_used == ctx->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    ctx->ev_pool.push_back(e);
  }
  return ctx->ev_pool[ctx->ev_used++];
}

struct Prof {
  ideq_ctx* ctx;
  int cls;
  double flops, bytes;
  cudaEvent_t a = nullptr;
  Prof(ideq_ctx* c, int k, double f = 0, double b = 0) : ctx(c), cls(k), flops(f), bytes(b) {
    if (ctx->counting) { ctx->cnt_flops[k] += f; ctx->cnt_bytes[k] += b; }
    if (ctx->segt) ctx->segt->enter(k == IDEQ_K_FIDELITY ? IDEQ_K_STEP : k);  // the step's passes count with it
    if (ctx->profiling) { a = next_event(ctx); cudaEventRecord(a, ctx->stream); }
  }
  ~Prof() {
    if (ctx->profiling) {
      cudaEvent_t b = next_event(ctx);
      cudaEventRecord(b, ctx->stream);
      ctx->pending.push_back({a, b, cls, flops, bytes});
    }
  }
};

void collect_profile(ideq_ctx* ctx) {
  if (ctx->pending.empty()) return;
  cudaStreamSynchronize(ctx->stream);
  for (auto& e : ctx->pending) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e.a, e.b);
    ctx->prof.ms[e.cls] += ms;
    ctx->prof.launches[e.cls] += 1;
    ctx->prof.flops[e.cls] += e.flops;
    ctx->prof.bytes[e.cls] += e.bytes;
  }
  ctx->pending.clear();
  ctx->ev_used = 0;
}

// `off` = first image of the micro-batch x (C*H*W): the head / tail layers read and write the
// solver's image planes of those images; every other layer works in the network workspace.
void run_layer(ideq_ctx* ctx, const Layer& L, long long off) {
  cudaStream_t s = ctx->stream;
  const bool bf = ctx->prec == IDEQ_PREC_BF16;
  auto sh = [off](const float* p) { return p ? p + off : p; };
  auto shw = [off](float* p) { return p ? p + off : p; };
  if (L.kind == L_RBF) {
    Prof p(ctx, IDEQ_K_CONV_TC, L.flops, L.bytes);
    rbf_launch(L.rbf, s);
  } else if (L.kind == L_IMG2FEAT_TC) {
    Prof p(ctx, IDEQ_K_HEADTAIL, L.flops, L.bytes);
    launch_img2feat_tc(L.i2f, sh(L.in_img), (const __nv_bfloat16*)L.wB, ctx->skip_frozen ? ctx->act_list : nullptr,
                       ctx->n_active,
                       L.N, L.C, L.H, L.W, L.wfeat, ctx->num_sms, s);
  } else if (L.kind == L_GEMM) {
    if (L.tc) {
      Prof p(ctx, L.headtail ? IDEQ_K_HEADTAIL : IDEQ_K_CONV_TC, L.flops, L.bytes);
      if (L.out_img) tc_plan_set_image(L.plan, shw(L.out_img), sh(L.aux_img), L.alpha, ctx->C);
      tc_launch(L.plan, s);
    } else {
      Prof p(ctx, IDEQ_K_CONV_SIMT, L.flops, L.bytes);
      if (bf)
        launch_conv_simt<__nv_bfloat16>(L.g, (const __nv_bfloat16*)L.in, (const __nv_bfloat16*)L.wB,
                                        (__nv_bfloat16*)L.out, (const __nv_bfloat16*)L.aux, s);
      else
        launch_conv_simt<float>(L.g, (const float*)L.in, (const float*)L.wB, (float*)L.out, (const float*)L.aux, s);
    }
  } else if (L.kind == L_IMG2FEAT) {
    Prof p(ctx, IDEQ_K_HEADTAIL, L.flops, L.bytes);
    if (bf)
      launch_img2feat<__nv_bfloat16>(sh(L.in_img), (const float*)L.wB, (__nv_bfloat16*)L.out,
                                     (const __nv_bfloat16*)L.aux, L.epi, L.N, L.C, L.H, L.W, L.wfeat, s);
    else
      launch_img2feat<float>(sh(L.in_img), (const float*)L.wB, (float*)L.out, (const float*)L.aux, L.epi, L.N, L.C,
                             L.H, L.W, L.wfeat, s);
  } else {
    Prof p(ctx, IDEQ_K_HEADTAIL, L.flops, L.bytes);
    if (bf)
      launch_feat2img<__nv_bfloat16>((const __nv_bfloat16*)L.in, (const float*)L.wB, shw(L.out_img), sh(L.aux_img),
                                     L.alpha, L.N, L.C, L.H, L.W, L.wfeat, s);
    else
      launch_feat2img<float>((const float*)L.in, (const float*)L.wB, shw(L.out_img), sh(L.aux_img), L.alpha, L.N,
                             L.C, L.H, L.W, L.wfeat, s);
  }
}

// Kernel-class filter of run_network: -1 = every layer (the iteration); otherwise only the layers
// of that ideq_kernel_class (class timing).
int layer_class(const Layer& L) {
  if (L.kind == L_RBF) return IDEQ_K_CONV_TC;
  if (L.kind == L_GEMM && L.tc && !L.headtail) return IDEQ_K_CONV_TC;
  if (L.kind == L_GEMM && !L.tc) return IDEQ_K_CONV_SIMT;
  return IDEQ_K_HEADTAIL;
}

// U_theta and its VJP for images [0, N): one pass of the program per micro-batch of <= mb images
// (the programs are built by prepare_programs before any capture).
void run_network(ideq_ctx* ctx, int N, int cls = -1) {
  const long long d = (long long)ctx->C * ctx->H * ctx->W;
  for (int first = 0; first < N; first += ctx->mb) {
    const int n = N - first < ctx->mb ? N - first : ctx->mb;
    const Program& P = ctx->progs.at(n);
    for (const auto& L : P.layers)
      if (cls < 0 || layer_class(L) == cls) run_layer(ctx, L, first * d);
  }
}

ideq_status prepare_programs(ideq_ctx* ctx, int N) {
  ideq_status st;
  const int n_full = N < ctx->mb ? N : ctx->mb;
  if ((st = build_program(ctx, n_full))) return st;
  if (N > ctx->mb && N % ctx->mb && (st = build_program(ctx, N % ctx->mb))) return st;
  return IDEQ_OK;
}

// The live-image list indexes images of the batch: used when one network pass covers the batch.
void enable_skip(ideq_ctx* ctx, bool on) {
  for (auto& kv : ctx->progs)
    for (auto& L : kv.second.layers) {
      if (L.plan) tc_plan_enable_skip(L.plan, on);
      if (L.rbf) rbf_enable_skip(L.rbf, on);
    }
}

// ------------------------------------------------------------------ fidelity + step
StepArgs make_step_args(ideq_ctx* ctx, int N, const float* y, float* x0, const ideq_params* p) {
  StepArgs a{};
  a.N = N; a.C = ctx->C; a.H = ctx->H; a.W = ctx->W;
  a.d = (long long)ctx->C * ctx->H * ctx->W;
  a.z = ctx->Z; a.zout = ctx->Z; a.gg = ctx->G; a.y = y;
  a.X0 = x0; a.X1 = ctx->X1;
  a.mask = ctx->d_mask; a.fbuf = ctx->fbuf; a.fbuf2 = ctx->fbuf2;
  a.kern = ctx->d_kern; a.ksize = ctx->op.ksize; a.kernel_per_image = ctx->op.kernel_per_image;
  if (p) { a.lam = p->lambda; a.tau = p->tau; a.beta = p->beta; }
  a.inv_s2 = ctx->op.kind == IDEQ_OP_RICIAN ? 1.f / (ctx->op.sigma * ctx->op.sigma) : 0.f;
  a.active = ctx->active; a.kdev = ctx->kdev; a.partials = ctx->partials;
  return a;
}

FftArgs make_fft_args(ideq_ctx* ctx, const float* y, const ideq_params* p) {
  FftArgs f{};
  f.C = ctx->C; f.H = ctx->H; f.W = ctx->W; f.J = ctx->op.n_phase;
  fft_fill_args(f);
  f.tw_h = ctx->tw_h; f.tw_w = ctx->tw_w; f.spec = ctx->spec;
  f.z = ctx->Z; f.gg = ctx->G; f.aty = ctx->fbuf2;
  if (p) { f.tau = p->tau; f.lam = p->lambda; }
  f.dgl = ctx->dgl; f.khat = ctx->khat; f.pmask = (const float2*)ctx->d_phase; f.y = y;
  f.active = ctx->active;
  return f;
}

int step_parts(ideq_ctx* ctx) {
  if (ctx->op.kind == IDEQ_OP_BLUR && ctx->op.blur_impl == IDEQ_BLUR_DIRECT && ctx->op.step == IDEQ_STEP_GRAD)
    return blur_parts_per_image(ctx->C, ctx->H, ctx->W, ctx->op.ksize);
  if ((ctx->op.kind == IDEQ_OP_BLUR || ctx->op.kind == IDEQ_OP_MRI) && ctx->op.step == IDEQ_STEP_PROX)
    return fft_parts_per_image(ctx->C, ctx->H, ctx->W);
  if (ctx->op.kind == IDEQ_OP_PHASE) return phase_parts_per_image(ctx->H, ctx->W, ctx->op.n_phase);
  const long long d = (long long)ctx->C * ctx->H * ctx->W;
  long long parts = d / 4096;
  if (parts < 1) parts = 1;
  if (parts > 256) parts = 256;
  return (int)parts;
}

void run_step(ideq_ctx* ctx, const StepArgs& a0) {
  StepArgs a = a0;
  a.parts = step_parts(ctx);
  cudaStream_t s = ctx->stream;
  const auto& op = ctx->op;
  if (op.kind == IDEQ_OP_INPAINT) {
    // reads z, grad g, x^k, y (fp32) and the u8 mask (one byte per pixel, shared by the C channels);
    // writes x^{k+1}, z^{k+1}
    Prof p(ctx, IDEQ_K_STEP, 0, (double)a.N * a.d * (24.0 + 1.0 / a.C));
    launch_pointwise_step(op.step == IDEQ_STEP_PROX ? STEP_PROX_INPAINT : STEP_GRAD_INPAINT, a, s);
  } else if (op.kind == IDEQ_OP_RICIAN) {
    Prof p(ctx, IDEQ_K_STEP, 0, (double)a.N * a.d * 4.0 * 6.0);
    launch_pointwise_step(STEP_GRAD_RICIAN, a, s);
  } else if (op.kind == IDEQ_OP_MRI && op.step == IDEQ_STEP_GRAD) {
    // F^-1 M F z through the half-spectrum passes, then x^{k+1} = z - tau(grad f + lam grad g)
    FftArgs f = make_fft_args(ctx, a.y, nullptr);
    f.dgl = ctx->mhalf;
    const double spec_b = (double)a.N * a.H * (a.W / 2 + 1) * 8.0;
    {
      Prof p(ctx, IDEQ_K_FIDELITY, 0, (double)a.N * a.d * 4.0 + 4.0 * spec_b);
      StepArgs dummy{};
      launch_blur_rows_fwd(f, ctx->Z, 0, a.N, s);
      launch_blur_cols(f, 0, a.N, s);
      launch_blur_rows_inv(f, dummy, ctx->fbuf, 0, a.N, s);
    }
    Prof p(ctx, IDEQ_K_STEP, 0, (double)a.N * a.d * 4.0 * 8.0);
    launch_pointwise_step(STEP_GRAD_MRI, a, s);
  } else if ((op.kind == IDEQ_OP_BLUR || op.kind == IDEQ_OP_MRI) && op.step == IDEQ_STEP_PROX) {
    // x^{k+1} = F^-1[ F(z - tau lam grad g + tau A^T y) / (1 + tau |K^|^2) ]   (prox P:80-84)
    FftArgs f = make_fft_args(ctx, a.y, nullptr);
    f.tau = a.tau; f.lam = a.lam;
    const double spec_b = (double)a.N * a.C * a.H * (a.W / 2 + 1) * 8.0;
    {
      Prof p(ctx, IDEQ_K_FIDELITY, 0, (double)a.N * a.d * 12.0 + spec_b);
      launch_blur_rows_fwd(f, nullptr, 1, a.N, s);
    }
    {
      Prof p(ctx, IDEQ_K_FIDELITY, 0, 2.0 * spec_b);
      launch_blur_cols(f, 0, a.N, s);
    }
    Prof p(ctx, IDEQ_K_STEP, 0, spec_b + (double)a.N * a.d * 4.0 * 3.0);
    launch_blur_rows_inv(f, a, nullptr, 1, a.N, s);
  } else if (op.kind == IDEQ_OP_BLUR) {
    {
      Prof p(ctx, IDEQ_K_FIDELITY, 2.0 * a.N * a.d * op.ksize * op.ksize, (double)a.N * a.d * 12.0);
      launch_blur_residual(a, s);
    }
    Prof p(ctx, IDEQ_K_STEP, 2.0 * a.N * a.d * op.ksize * op.ksize, (double)a.N * a.d * 4.0 * 6.0);
    launch_blur_adjoint(1, a, ctx->fbuf, s);
  } else if (op.kind == IDEQ_OP_PHASE) {
    // grad f = sum_j 2 Re(conj(D_j) F^-1[(|u_j|^2 - y_j) u_j]), x^{k+1} = z - tau(grad f + lam grad g)
    FftArgs f = make_fft_args(ctx, a.y, nullptr);
    f.tau = a.tau; f.lam = a.lam;
    const double spec_b = (double)a.N * op.n_phase * a.H * a.W * 8.0;
    {
      Prof p(ctx, IDEQ_K_FIDELITY, 0, (double)a.N * a.d * 4.0 + spec_b);
      launch_phase_rows_fwd(f, a.N, s);
    }
    {
      Prof p(ctx, IDEQ_K_FIDELITY, 0, 2.0 * spec_b + (double)a.N * op.n_phase * a.H * a.W * 4.0);
      launch_phase_cols(f, a.N, s);
    }
    Prof p(ctx, IDEQ_K_STEP, 0, spec_b + (double)a.N * a.d * 4.0 * 5.0);
    launch_phase_rows_inv(f, a, nullptr, 1, a.N, s);
  }
}

// Per-solve operator constants: A^T y (FFT) and the diagonal 1 / (1 + tau |K^|^2).
// MRI constants of a solve: fbuf2 = Re F^-1(M y) (the A^T y of the k-space prox and gradient),
// mhalf = M and dgl = 1 / (1 + tau M) on the half spectrum.
void prepare_mri(ideq_ctx* ctx, const float* y, float tau, int N) {
  FftArgs f = make_fft_args(ctx, y, nullptr);
  f.active = nullptr;
  StepArgs dummy{};
  launch_mri_fill(y, ctx->d_kmask, ctx->spec, N, ctx->H, ctx->W, sqrtf((float)ctx->H * (float)ctx->W), ctx->stream);
  launch_blur_cols(f, 3, N, ctx->stream);
  launch_blur_rows_inv(f, dummy, ctx->fbuf2, 0, N, ctx->stream);
  launch_mri_masks(ctx->d_kmask, ctx->mhalf, ctx->dgl, tau, ctx->H, ctx->W, ctx->stream);
}

void prepare_blur_prox(ideq_ctx* ctx, const float* y, float tau, int N) {
  FftArgs f = make_fft_args(ctx, y, nullptr);
  f.active = nullptr;
  StepArgs dummy{};
  launch_blur_rows_fwd(f, y, 0, N, ctx->stream);
  launch_blur_cols(f, 1, N, ctx->stream);
  launch_blur_rows_inv(f, dummy, ctx->fbuf2, 0, N, ctx->stream);
  launch_blur_diag(ctx->khat, tau, ctx->dgl, ctx->H * (ctx->W / 2 + 1), ctx->stream);
}

FinalizeArgs make_fin(ideq_ctx* ctx, int N, const ideq_params* p) {
  FinalizeArgs f{};
  f.N = N;
  f.parts = step_parts(ctx);
  f.check_every = p ? p->check_every : 1;
  f.stop_rule = p ? (int)p->stop_rule : 0;
  f.tol = p ? p->tol : 0.f;
  f.partials = ctx->partials;
  f.active = ctx->active; f.status = ctx->status; f.iters = ctx->iters;
  f.res = ctx->res; f.r_now = ctx->r_now; f.trace = ctx->trace; f.trace_cap = ctx->trace_cap; f.rmax = ctx->rmax;
  f.n_active = ctx->n_active; f.kdev = ctx->kdev; f.act_list = ctx->act_list;
  const bool next1 = p && (p->restart || p->averaging);
  f.restart = p ? p->restart : 0;
  f.B2 = p ? (double)p->restart_B * (double)p->restart_B : 0.0;
  f.averaging = p ? p->averaging : 0;
  f.K = p ? p->max_iter : 0;
  f.rk = ctx->rk; f.rsum = ctx->rsum; f.nrest = ctx->nrest; f.best = ctx->best; f.k0 = ctx->k0;
  f.flags = next1 ? ctx->flags : nullptr;  // null: the plain path pays nothing for NEXT-1
  return f;
}

// One iteration: network (forward + VJP), fidelity + update + partials, finalize, advance.
ideq_status enqueue_iteration(ideq_ctx* ctx, const StepArgs& a, const FinalizeArgs& f, bool with_allreduce) {
  run_network(ctx, a.N);
  run_step(ctx, a);
  {
    Prof p(ctx, IDEQ_K_REDUCE);
    launch_finalize(f, ctx->stream);
    if (f.flags) {  // restart (z^{k+1} := x^{k+1}) and averaging bookkeeping
      PostArgs pa{};
      pa.N = f.N; pa.d = a.d; pa.flags = f.flags; pa.kdev = f.kdev; pa.X0 = a.X0; pa.X1 = a.X1; pa.Z = ctx->Z;
      pa.Zsum = f.averaging ? ctx->Zsum : nullptr;
      pa.Xsnap = ctx->Xsnap;
      launch_post_step(pa, ctx->stream);
    }
    launch_advance_a(f, ctx->stream);
    if (with_allreduce && ctx->comm) {
      int r = g_nccl.AllReduce(ctx->rmax, ctx->rmax, 1, NCCL_FLOAT32, NCCL_MAX, ctx->comm, ctx->stream);
      if (r != 0) return fail(ctx, IDEQ_E_NCCL, "ncclAllReduce failed: %s", g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?");
    }
    launch_advance_b(f, ctx->stream);
  }
  return IDEQ_OK;
}

ideq_status check_ctx(ideq_ctx* ctx) {
  if (!ctx) return IDEQ_E_INVALID;
  if (ctx->poisoned) return fail(ctx, IDEQ_E_STATE, "context poisoned by an earlier CUDA/NCCL error: %s", ctx->err.c_str());
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return fail(ctx, IDEQ_E_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
  return IDEQ_OK;
}

ideq_status validate_params(ideq_ctx* ctx, int batch, const ideq_params* p) {
  if (!p) return fail(ctx, IDEQ_E_INVALID, "params is NULL");
  if (batch < 1 || batch > ctx->maxN) return fail(ctx, IDEQ_E_INVALID, "batch %d outside [1, %d]", batch, ctx->maxN);
  if (!(p->tau > 0.f) || !(p->lambda >= 0.f) || !(p->beta >= 0.f && p->beta < 1.f) || p->max_iter < 1 ||
      !(p->tol >= 0.f) || p->check_every < 1 || (p->stop_rule != IDEQ_STOP_PER_IMAGE && p->stop_rule != IDEQ_STOP_GLOBAL_MAX))
    return fail(ctx, IDEQ_E_INVALID, "invalid params (tau>0, lambda>=0, 0<=beta<1, max_iter>=1, tol>=0, check_every>=1)");
  if (p->restart < 0 || p->restart > 2 || (p->restart && !(p->restart_B >= 0.f)))
    return fail(ctx, IDEQ_E_INVALID, "restart must be 0, 1 (Alg. 1) or 2 (Alg. 2) with restart_B >= 0");
  if (p->averaging != 0 && p->averaging != 1) return fail(ctx, IDEQ_E_INVALID, "averaging must be 0 or 1");
  if (p->averaging && p->tol != 0.f)
    return fail(ctx, IDEQ_E_INVALID, "averaging (Alg. 1 steps 12-13) needs a fixed iteration count: tol = 0");
  if (!ctx->op_set) return fail(ctx, IDEQ_E_STATE, "ideq_set_operator must be called before solving");
  // the operator's per-image data (kernels, masks) and its FFT work spectrum are sized for the
  // batch given to ideq_set_operator
  if (batch > ctx->op_batch)
    return fail(ctx, IDEQ_E_INVALID, "batch %d exceeds the operator's batch %d", batch, ctx->op_batch);
  if (p->compute_frozen != 0 && p->compute_frozen != 1) return fail(ctx, IDEQ_E_INVALID, "compute_frozen must be 0 or 1");
  return IDEQ_OK;
}

ideq_status operator_runnable(ideq_ctx* ctx) {
  const auto& op = ctx->op;
  if (op.kind == IDEQ_OP_PHASE && op.step == IDEQ_STEP_PROX)
    return fail(ctx, IDEQ_E_UNSUPPORTED, "phase retrieval has no closed-form prox (cf. PAPER l.1079)");
  if (op.kind == IDEQ_OP_RICIAN && op.step == IDEQ_STEP_PROX)
    return fail(ctx, IDEQ_E_UNSUPPORTED, "the Rician fidelity has no closed-form prox (PAPER l.1079)");
  if (op.kind == IDEQ_OP_BLUR && op.step == IDEQ_STEP_GRAD && op.blur_impl == IDEQ_BLUR_FFT)
    return fail(ctx, IDEQ_E_UNSUPPORTED, "the blur gradient step uses the direct convolution (blur_impl DIRECT)");
  return IDEQ_OK;
}

ideq_status finish_solve(ideq_ctx* ctx, float* x, int N, const ideq_params* p, ideq_image_stat* stats,
                         float* trace_host, bool next1);

// The whole solve of a tiny-network deblurring problem (BASELINE C1) fits one persistent kernel per
// image (tiny_solve.cu): no per-iteration launches. Eligible: TINY3 with hidden width 16, C = 1,
// identity skip, softplus, fp32, direct blur gradient step, per-image stop, no restart /
// averaging, not profiling.
bool tiny_fused_ok(ideq_ctx* ctx, const ideq_params* p) {
  const auto& n = ctx->net;
  const auto& op = ctx->op;
  return n.arch == IDEQ_NET_TINY3 && n.widths[0] == 16 && ctx->C == 1 && n.identity_skip &&
         n.act == IDEQ_ACT_SOFTPLUS && ctx->prec == IDEQ_PREC_FP32 && op.kind == IDEQ_OP_BLUR &&
         op.step == IDEQ_STEP_GRAD && op.blur_impl == IDEQ_BLUR_DIRECT && p->stop_rule == IDEQ_STOP_PER_IMAGE &&
         !p->restart && !p->averaging && !ctx->profiling && tiny_solve_supported(ctx->H, ctx->W, op.ksize);
}

ideq_status launch_tiny_fused(ideq_ctx* ctx, const float* y, float* x, int N, const ideq_params* p) {
  if (!ctx->wdev.count("tiny#blob")) {  // the fp32 blob (c1, c2, c3 in blob order), uploaded once
    ideq_status st = upload_f32(ctx, "tiny#blob", ctx->blob);
    if (st) return st;
  }
  const float* wb = (const float*)ctx->wdev["tiny#blob"];
  const int w = 16, C = 1;
  TinySolveArgs a{};
  a.N = N; a.H = ctx->H; a.W = ctx->W; a.ks = ctx->op.ksize; a.kper = ctx->op.kernel_per_image;
  a.kern = ctx->d_kern;
  a.w1 = wb; a.w2 = wb + w * C * 9; a.w3 = wb + w * C * 9 + w * w * 9;
  a.y = y; a.x = x;
  a.lam = p->lambda; a.tau = p->tau; a.beta = p->beta; a.tol = p->tol;
  a.max_iter = p->max_iter; a.check_every = p->check_every;
  a.iters = ctx->iters; a.res = ctx->res; a.status = ctx->status;
  a.trace = ctx->trace; a.trace_cap = ctx->trace_cap; a.kdone = ctx->kdev;
  CK(cudaMemsetAsync(ctx->trace, 0, sizeof(float) * ctx->trace_cap, ctx->stream));
  CK(cudaMemsetAsync(ctx->kdev, 0, sizeof(int), ctx->stream));
  launch_tiny_solve(a, ctx->stream);
  CK(cudaGetLastError());
  return IDEQ_OK;
}

ideq_status solve_device(ideq_ctx* ctx, const float* y, float* x, int N, const ideq_params* p,
                         ideq_image_stat* stats, float* trace_host) {
  ideq_status st;
  if ((st = validate_params(ctx, N, p))) return st;
  if ((st = operator_runnable(ctx))) return st;
  if (!y || !x || !stats) return fail(ctx, IDEQ_E_INVALID, "NULL y/x/stats");
  const bool fused = tiny_fused_ok(ctx, p);
  ctx->last_fused = fused;
  if (fused) {
    ctx->have_last = true;
    ctx->last_N = N;
    if ((st = launch_tiny_fused(ctx, y, x, N, p))) return st;
    return finish_solve(ctx, x, N, p, stats, trace_host, false);
  }
  if ((st = prepare_programs(ctx, N))) return st;
  const long long d = (long long)ctx->C * ctx->H * ctx->W;
  cudaStream_t s = ctx->stream;
  // x^{-1} = x^0; z^0 = x^0
  CK(cudaMemcpyAsync(ctx->X1, x, sizeof(float) * N * d, cudaMemcpyDeviceToDevice, s));
  CK(cudaMemcpyAsync(ctx->Z, x, sizeof(float) * N * d, cudaMemcpyDeviceToDevice, s));
  if (p->averaging) CK(cudaMemcpyAsync(ctx->Zsum, x, sizeof(float) * N * d, cudaMemcpyDeviceToDevice, s));  // z^0
  FinalizeArgs f = make_fin(ctx, N, p);
  if (f.parts > ctx->parts_cap) return fail(ctx, IDEQ_E_INVALID, "internal: partial buffer too small");
  launch_init_state(f, s);
  if (ctx->op.kind == IDEQ_OP_BLUR && ctx->op.step == IDEQ_STEP_PROX) prepare_blur_prox(ctx, y, p->tau, N);
  if (ctx->op.kind == IDEQ_OP_MRI) prepare_mri(ctx, y, p->tau, N);
  StepArgs a = make_step_args(ctx, N, y, x, p);
  // skip frozen images' tiles only when images can freeze early and one network pass covers the
  // batch (the live list indexes the batch)
  ctx->skip_frozen = p->tol > 0.f && p->stop_rule == IDEQ_STOP_PER_IMAGE && !p->compute_frozen && N <= ctx->mb;
  enable_skip(ctx, ctx->skip_frozen);
  ctx->have_last = true;
  ctx->last_N = N;
  ctx->last_a = a;
  ctx->last_f = f;
  const bool global = p->stop_rule == IDEQ_STOP_GLOBAL_MAX;
  const bool poll = p->tol > 0.f;
  const int poll_every = global ? p->check_every : 4;
  if (ctx->profiling) {
    for (int k = 0; k < p->max_iter; ++k) {
      const bool chk = global && ((k + 1) % p->check_every == 0);
      if ((st = enqueue_iteration(ctx, a, f, chk))) return st;
      if (poll && ((k + 1) % poll_every == 0)) {
        CK(cudaMemcpyAsync(ctx->h_pinned, ctx->n_active, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (*ctx->h_pinned == 0) break;
      }
    }
    collect_profile(ctx);
  } else {
    // capture one iteration (plain and with the convergence all-reduce)
    char keybuf[256];
    // every value the captured kernels hold by value: the pointers, the step parameters and the
    // finalize arguments (max_iter sets the averaging window K, compute_frozen the tile lists)
    snprintf(keybuf, sizeof(keybuf), "%p|%p|%d|%a|%a|%a|%a|%d|%d|%d|%a|%d|%d|%d", (const void*)y, (void*)x, N,
             p->lambda, p->tau, p->beta, p->tol, p->check_every, (int)p->stop_rule, p->restart, p->restart_B,
             p->averaging, p->max_iter, p->compute_frozen);
    if (ctx->graph_key != keybuf) {
      if (ctx->gexec_plain) { cudaGraphExecDestroy(ctx->gexec_plain); ctx->gexec_plain = nullptr; }
      if (ctx->gexec_check) { cudaGraphExecDestroy(ctx->gexec_check); ctx->gexec_check = nullptr; }
      for (int v = 0; v < 2; ++v) {
        if (v == 1 && !(global && ctx->comm)) break;
        cudaGraph_t graph;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        ideq_status st2 = enqueue_iteration(ctx, a, f, v == 1);
        cudaError_t ec = cudaStreamEndCapture(s, &graph);
        if (st2) return st2;
        if (ec != cudaSuccess) return fail(ctx, IDEQ_E_CUDA, "graph capture: %s", cudaGetErrorString(ec));
        cudaGraphExec_t ge;
        CK(cudaGraphInstantiate(&ge, graph, 0));
        cudaGraphDestroy(graph);
        (v == 0 ? ctx->gexec_plain : ctx->gexec_check) = ge;
      }
      ctx->graph_key = keybuf;
    }
    for (int k = 0; k < p->max_iter; ++k) {
      const bool chk = global && ctx->comm && ((k + 1) % p->check_every == 0);
      CK(cudaGraphLaunch(chk ? ctx->gexec_check : ctx->gexec_plain, s));
      if (poll && ((k + 1) % poll_every == 0) && k + 1 < p->max_iter) {
        CK(cudaMemcpyAsync(ctx->h_pinned, ctx->n_active, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (*ctx->h_pinned == 0) break;
      }
    }
  }
  launch_gather(ctx->iters, ctx->X1, x, N, d, s);
  if (p->averaging) launch_avg_out(ctx->k0, ctx->status, ctx->iters, p->max_iter, ctx->Xsnap, x, N, d, s);
  return finish_solve(ctx, x, N, p, stats, trace_host, true);
}

// Per-image statistics and the trace back to the host; IDEQ_E_DIVERGED if any image diverged.
ideq_status finish_solve(ideq_ctx* ctx, float* x, int N, const ideq_params* p, ideq_image_stat* stats,
                         float* trace_host, bool next1) {
  (void)x;
  cudaStream_t s = ctx->stream;
  std::vector<int> it(N), stv(N), nr(N, 0), k0v(N, -1);
  if (next1 && p->restart) CK(cudaMemcpyAsync(nr.data(), ctx->nrest, sizeof(int) * N, cudaMemcpyDeviceToHost, s));
  if (next1 && p->averaging) CK(cudaMemcpyAsync(k0v.data(), ctx->k0, sizeof(int) * N, cudaMemcpyDeviceToHost, s));
  std::vector<float> rs(N);
  CK(cudaMemcpyAsync(it.data(), ctx->iters, sizeof(int) * N, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(stv.data(), ctx->status, sizeof(int) * N, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(rs.data(), ctx->res, sizeof(float) * N, cudaMemcpyDeviceToHost, s));
  if (trace_host) {
    const int nt = p->max_iter < ctx->trace_cap ? p->max_iter : ctx->trace_cap;
    // iterations that never ran report NaN
    std::vector<float> tr(nt);
    CK(cudaMemcpyAsync(tr.data(), ctx->trace, sizeof(float) * nt, cudaMemcpyDeviceToHost, s));
    int kdone = 0;
    CK(cudaMemcpyAsync(&kdone, ctx->kdev, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int k = 0; k < p->max_iter; ++k) trace_host[k] = (k < nt && k < kdone) ? tr[k] : NAN;
  }
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  bool diverged = false;
  for (int i = 0; i < N; ++i) {
    stats[i].iters = it[i];
    stats[i].residual = rs[i];
    stats[i].status = stv[i];
    stats[i].restarts = nr[i];
    // K0 only where x-hat IS the average (same condition as avg_out_kernel)
    stats[i].k0 = (p->averaging && stv[i] != 2 && it[i] == p->max_iter) ? k0v[i] : -1;
    if (stv[i] == 2) diverged = true;
  }
  if (diverged) return fail(ctx, IDEQ_E_DIVERGED, "at least one image produced a non-finite iterate");
  return IDEQ_OK;
}

}  // namespace

namespace ideq {
void init_kernel_attributes() {
  static bool done = false;
  if (done) return;
  init_attrs_simt();
  init_attrs_tc();
  init_attrs_step();
  init_attrs_fft();
  init_attrs_tiny();
  init_attrs_rbf();
  done = true;
}
}  // namespace ideq

// ======================================================================== C ABI
extern "C" {

int ideq_abi_version(void) { return IDEQ_ABI_VERSION; }

const char* ideq_last_error(const ideq_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

ideq_status ideq_get_nccl_id(unsigned char out[128]) {
  if (!out) return IDEQ_E_INVALID;
  std::string err;
  if (!g_nccl.load(err)) return IDEQ_E_NCCL;
  nccl_uid id;
  if (g_nccl.GetUniqueId(&id) != 0) return IDEQ_E_NCCL;
  memcpy(out, &id, 128);
  return IDEQ_OK;
}

ideq_status ideq_create(const ideq_net_desc* net, ideq_precision prec, int device, void* cuda_stream, int max_batch,
                        int H, int W, const ideq_dist* dist, ideq_ctx** out) {
  return ideq_create_ex(net, prec, device, cuda_stream, max_batch, H, W, dist, nullptr, out);
}

ideq_status ideq_get_plan(const ideq_ctx* ctx, int* micro_batch, size_t* workspace_bytes) {
  if (!ctx) return IDEQ_E_INVALID;
  if (micro_batch) *micro_batch = ctx->mb;
  if (workspace_bytes) *workspace_bytes = ctx->net_bytes;
  return IDEQ_OK;
}

ideq_status ideq_create_ex(const ideq_net_desc* net, ideq_precision prec, int device, void* cuda_stream, int max_batch,
                           int H, int W, const ideq_dist* dist, const ideq_plan_opts* opts, ideq_ctx** out) {
  if (!net || !out || !net->weights) return IDEQ_E_INVALID;
  *out = nullptr;
  std::unique_ptr<ideq_ctx> holder(new ideq_ctx());
  ideq_ctx* ctx = holder.get();
  ctx->net = *net;
  ctx->prec = prec;
  ctx->device = device;
  ctx->stream = (cudaStream_t)cuda_stream;
  ctx->maxN = max_batch;
  ctx->H = H;
  ctx->W = W;
  ctx->C = net->channels;
  ctx->elt = prec == IDEQ_PREC_BF16 ? 2 : 4;
  if (prec != IDEQ_PREC_FP32 && prec != IDEQ_PREC_BF16) return IDEQ_E_INVALID;
  if (max_batch < 1 || H < 1 || W < 1 || !(net->channels == 1 || net->channels == 3)) return IDEQ_E_INVALID;
  WeightSlices ws;
  size_t total = 0;
  if (net->arch == IDEQ_NET_TINY3) {
    const int w = net->widths[0];
    if (!(w == 16 || w == 32 || w == 64)) return IDEQ_E_INVALID;
  } else if (net->arch == IDEQ_NET_UNET4) {
    if (H % 8 || W % 8 || net->res_blocks < 1) return IDEQ_E_INVALID;
    if (!(net->widths[0] == 32 || net->widths[0] == 64)) return IDEQ_E_INVALID;
    for (int l = 0; l < 4; ++l)
      if (net->widths[l] < 16 || net->widths[l] % 16) return IDEQ_E_INVALID;
    if (prec == IDEQ_PREC_BF16)
      for (int l = 0; l < 4; ++l)
        if (net->widths[l] % 32) return IDEQ_E_INVALID;
  } else {
    return IDEQ_E_INVALID;
  }
  slice_weights(*net, ws, total);
  if (total != net->n_weights) return IDEQ_E_INVALID;
  ctx->blob.assign(net->weights, net->weights + total);
  ctx->net.weights = nullptr;

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    *out = holder.release();
    return fail(*out, IDEQ_E_CUDA, "no CUDA device available (this library has no CPU fallback)");
  }
  cudaDeviceProp prop;
  if (cudaSetDevice(device) != cudaSuccess || cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
    *out = holder.release();
    return fail(*out, IDEQ_E_CUDA, "cannot use device %d", device);
  }
  if (prop.major != 10) {
    *out = holder.release();
    return fail(*out, IDEQ_E_CUDA, "device %d is sm_%d%d; this library is built for sm_100a only", device, prop.major,
                prop.minor);
  }
  ctx->num_sms = prop.multiProcessorCount;
  init_kernel_attributes();
  if (!ctx->stream) {
    // graph capture is not allowed on the legacy default stream: own a stream instead
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
      *out = holder.release();
      return fail(*out, IDEQ_E_CUDA, "cannot create a stream");
    }
    ctx->own_stream = true;
  }

  // ---- solver state (every image of a solve)
  const int N = max_batch;
  ideq_status st;
  const size_t plane = (size_t)N * ctx->C * H * W * sizeof(float);
  void* p;
#define AL(field, bytes)                                                          \
  if ((st = dalloc(ctx, &p, (bytes)))) { *out = holder.release(); return st; } \
  ctx->field = (decltype(ctx->field))p;
  AL(X1, plane) AL(Z, plane) AL(G, plane) AL(Hc, plane) AL(fbuf, plane) AL(fbuf2, plane)
  {  // residual partials per image: the largest count any fidelity/step kernel can produce at this size
    int pc = 256;
    const int cand[3] = {blur_parts_per_image(ctx->C, H, W, 0) /* 32-pixel tiles: the larger count */, fft_parts_per_image(ctx->C, H, W),
                         phase_parts_per_image(H, W, 16) /* the most masks the register pass takes */};
    for (int v : cand) pc = v > pc ? v : pc;
    ctx->parts_cap = pc;
  }
  AL(partials, (size_t)N * ctx->parts_cap * 3 * sizeof(float))
  AL(active, N * sizeof(int)) AL(status, N * sizeof(int)) AL(iters, N * sizeof(int)) AL(act_list, N * sizeof(int))
  AL(rk, N * sizeof(int)) AL(rsum, N * sizeof(double)) AL(flags, N * sizeof(int)) AL(nrest, N * sizeof(int))
  AL(best, N * sizeof(float)) AL(k0, N * sizeof(int)) AL(Zsum, plane) AL(Xsnap, plane)
  AL(res, N * sizeof(float)) AL(r_now, N * sizeof(float)) AL(rmax, 16) AL(n_active, 16) AL(kdev, 16)
  AL(trace, ctx->trace_cap * sizeof(float))
#undef AL
  if (cudaMallocHost(&ctx->h_pinned, 64) != cudaSuccess) { *out = holder.release(); return fail(*out, IDEQ_E_NOMEM, "pinned alloc"); }
  cudaMemset(ctx->trace, 0xff, ctx->trace_cap * sizeof(float));

  // ---- workspace plan: the network's activations (work buffers + saved activations of every
  // residual block) for a micro-batch of mb images; a solve runs the network once per micro-batch
  // (C5's 512 images need ~221 GB of activations in bf16, beyond one GPU)
  size_t per_img = 0;  // network workspace bytes per image
  if (net->arch == IDEQ_NET_TINY3) {
    per_img = (size_t)4 * H * W * net->widths[0] * ctx->elt;
  } else {
    for (int l = 0; l < 4; ++l)
      per_img += (size_t)(3 + net->res_blocks + (l < 3 ? net->res_blocks : 0)) * (H >> l) * (W >> l) * net->widths[l] * ctx->elt;
  }
  {
    int mb = opts ? opts->micro_batch : 0;
    if (mb < 0) { *out = holder.release(); return fail(*out, IDEQ_E_INVALID, "micro_batch must be >= 0"); }
    if (mb == 0) {
      size_t budget = opts ? opts->workspace_bytes : 0;
      if (budget == 0) {
        size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) { cudaGetLastError(); fr = 0; }
        // kept free for what set_operator / solve_host allocate later (operator data, FFT work
        // spectrum, host staging of y and x) and for the runtime: 2 GB + 3 fp32 planes per image
        const size_t reserve = ((size_t)2 << 30) + 3 * plane;
        budget = fr > reserve ? (size_t)((double)(fr - reserve) * 0.9) : 0;
      }
      mb = (int)std::min<size_t>((size_t)N, budget / (per_img ? per_img : 1));
      if (mb < 1) {
        *out = holder.release();
        return fail(*out, IDEQ_E_NOMEM, "network workspace of one image (%zu bytes) exceeds the budget (%zu bytes)",
                    per_img, budget);
      }
    }
    if (mb > N) mb = N;
    const int nmb = (N + mb - 1) / mb;  // balanced micro-batches
    ctx->mb = (N + nmb - 1) / nmb;
    ctx->net_bytes = per_img * ctx->mb;
  }
  const int M = ctx->mb;
  if (net->arch == IDEQ_NET_TINY3) {
    const size_t e = (size_t)M * H * W * net->widths[0] * ctx->elt;
    ctx->lvl_buf.assign(1, std::vector<void*>(3, nullptr));
    for (int i = 0; i < 2; ++i) if ((st = dalloc(ctx, &ctx->lvl_buf[0][i], e))) { *out = holder.release(); return st; }
    void* a1; void* a2;
    if ((st = dalloc(ctx, &a1, e)) || (st = dalloc(ctx, &a2, e))) { *out = holder.release(); return st; }
    ctx->saved["a1"] = a1;
    ctx->saved["a2"] = a2;
  } else {
    ctx->lvl_buf.assign(4, std::vector<void*>(3, nullptr));
    for (int l = 0; l < 4; ++l) {
      const size_t e = (size_t)M * (H >> l) * (W >> l) * net->widths[l] * ctx->elt;
      for (int i = 0; i < 3; ++i) if ((st = dalloc(ctx, &ctx->lvl_buf[l][i], e))) { *out = holder.release(); return st; }
      for (int r = 0; r < net->res_blocks; ++r) {
        void* a;
        if ((st = dalloc(ctx, &a, e))) { *out = holder.release(); return st; }
        ctx->saved["e" + std::to_string(l) + "." + std::to_string(r)] = a;
        if (l < 3) {
          if ((st = dalloc(ctx, &a, e))) { *out = holder.release(); return st; }
          ctx->saved["d" + std::to_string(l) + "." + std::to_string(r)] = a;
        }
      }
    }
  }

  // ---- distribution
  if (dist && dist->world >= 1) {
    std::string err;
    if (!g_nccl.load(err)) { *out = holder.release(); return fail(*out, IDEQ_E_NCCL, "%s", err.c_str()); }
    nccl_uid id;
    memcpy(&id, dist->nccl_id, 128);
    int r = g_nccl.CommInitRank(&ctx->comm, dist->world, id, dist->rank);
    if (r != 0) { *out = holder.release(); return fail(*out, IDEQ_E_NCCL, "ncclCommInitRank failed (%d)", r); }
    ctx->rank = dist->rank;
    ctx->world = dist->world;
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { *out = holder.release(); return fail(*out, IDEQ_E_CUDA, "create: %s", cudaGetErrorString(e)); }
  *out = holder.release();
  return IDEQ_OK;
}

}  // extern "C"

namespace {
// Twiddle tables (fp64 -> fp32, constant setup) and the work spectrum of the FFT operators.
ideq_status setup_fft(ideq_ctx* ctx, size_t spec_elems) {
  const int H = ctx->H, W = ctx->W;
  if (!fft_size_ok(H, W)) return fail(ctx, IDEQ_E_UNSUPPORTED, "FFT operators need power-of-two H, W in [4, 1024]");
  ideq_status st;
  void* p;
  for (int which = 0; which < 2; ++which) {
    const int n = which == 0 ? H : W;
    std::vector<float2> tw(n / 2);
    for (int k = 0; k < n / 2; ++k) {
      const double a = -2.0 * M_PI * (double)k / (double)n;
      tw[k] = make_float2((float)cos(a), (float)sin(a));
    }
    if ((st = dalloc(ctx, &p, sizeof(float2) * (n / 2 > 0 ? n / 2 : 1)))) return st;
    CK(cudaMemcpy(p, tw.data(), sizeof(float2) * tw.size(), cudaMemcpyHostToDevice));
    (which == 0 ? ctx->tw_h : ctx->tw_w) = (float2*)p;
  }
  if ((st = dalloc(ctx, &p, sizeof(float2) * spec_elems))) return st;
  ctx->spec = (float2*)p;
  return IDEQ_OK;
}
}  // namespace

extern "C" {

ideq_status ideq_set_operator(ideq_ctx* ctx, const ideq_operator_desc* op, int batch) {
  ideq_status st;
  if ((st = check_ctx(ctx))) return st;
  if (!op || batch < 1 || batch > ctx->maxN) return fail(ctx, IDEQ_E_INVALID, "bad operator or batch");
  const int H = ctx->H, W = ctx->W;
  if (op->kind == IDEQ_OP_BLUR) {
    if (!op->kernels || op->ksize < 1 || op->ksize % 2 == 0 || op->ksize > 63)
      return fail(ctx, IDEQ_E_INVALID, "blur needs an odd ksize <= 63 and kernels");
    if (op->step == IDEQ_STEP_PROX && op->blur_impl != IDEQ_BLUR_FFT)
      return fail(ctx, IDEQ_E_INVALID, "the blur prox needs blur_impl = FFT");
    const size_t n = (size_t)(op->kernel_per_image ? batch : 1) * op->ksize * op->ksize;
    void* p;
    if ((st = dalloc(ctx, &p, n * 4))) return st;
    CK(cudaMemcpy(p, op->kernels, n * 4, cudaMemcpyHostToDevice));
    ctx->d_kern = (float*)p;
    if (op->blur_impl == IDEQ_BLUR_FFT) {
      if (op->kernel_per_image) return fail(ctx, IDEQ_E_UNSUPPORTED, "FFT blur needs one kernel shared by the batch");
      if (op->ksize > H || op->ksize > W) return fail(ctx, IDEQ_E_INVALID, "kernel larger than the image");
      if ((st = setup_fft(ctx, (size_t)batch * ctx->C * H * (W / 2 + 1)))) return st;
      // K^ = 2-D DFT of the kernel embedded with its centre tap at the origin (computed on device)
      void* q;
      if ((st = dalloc(ctx, &q, sizeof(float2) * H * (W / 2 + 1)))) return st;
      ctx->khat = (float2*)q;
      if ((st = dalloc(ctx, &q, sizeof(float) * H * (W / 2 + 1)))) return st;
      ctx->dgl = (float*)q;
      launch_embed_kernel(ctx->d_kern, op->ksize, ctx->fbuf, H, W, ctx->stream);
      FftArgs f = make_fft_args(ctx, nullptr, nullptr);
      f.C = 1;
      f.active = nullptr;
      launch_blur_rows_fwd(f, ctx->fbuf, 0, 1, ctx->stream);
      launch_blur_cols(f, 2, 1, ctx->stream);
      CK(cudaMemcpyAsync(ctx->khat, ctx->spec, sizeof(float2) * H * (W / 2 + 1), cudaMemcpyDeviceToDevice,
                         ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      CK(cudaGetLastError());
    }
  } else if (op->kind == IDEQ_OP_INPAINT) {
    if (!op->masks) return fail(ctx, IDEQ_E_INVALID, "inpainting needs masks");
    void* p;
    if ((st = dalloc(ctx, &p, (size_t)batch * H * W))) return st;
    CK(cudaMemcpy(p, op->masks, (size_t)batch * H * W, cudaMemcpyHostToDevice));
    ctx->d_mask = (uint8_t*)p;
  } else if (op->kind == IDEQ_OP_PHASE) {
    if (ctx->C != 1) return fail(ctx, IDEQ_E_INVALID, "phase retrieval needs C = 1");
    if (op->step == IDEQ_STEP_PROX) return fail(ctx, IDEQ_E_UNSUPPORTED, "no closed-form prox for phase retrieval");
    if (!op->phase_masks || op->n_phase < 1) return fail(ctx, IDEQ_E_INVALID, "phase retrieval needs phase masks");
    void* p;
    const size_t n = (size_t)op->n_phase * H * W * 2;
    if ((st = dalloc(ctx, &p, n * 4))) return st;
    CK(cudaMemcpy(p, op->phase_masks, n * 4, cudaMemcpyHostToDevice));
    ctx->d_phase = (float*)p;
    if ((st = setup_fft(ctx, (size_t)batch * op->n_phase * H * W))) return st;
  } else if (op->kind == IDEQ_OP_MRI) {
    if (ctx->C != 1) return fail(ctx, IDEQ_E_INVALID, "MRI needs C = 1 (real magnitude image, zero phase)");
    if (!op->masks) return fail(ctx, IDEQ_E_INVALID, "MRI needs a k-space mask [H][W]");
    for (int ky = 0; ky < H; ++ky)  // reading R7: the k-space prox is the real-image prox only then
      for (int kx = 0; kx < W; ++kx)
        if ((op->masks[ky * W + kx] != 0) != (op->masks[((H - ky) % H) * W + (W - kx) % W] != 0))
          return fail(ctx, IDEQ_E_INVALID, "MRI mask must be Hermitian-symmetric (M[-ky][-kx] == M[ky][kx])");
    void* p;
    if ((st = dalloc(ctx, &p, (size_t)H * W))) return st;
    CK(cudaMemcpy(p, op->masks, (size_t)H * W, cudaMemcpyHostToDevice));
    ctx->d_kmask = (uint8_t*)p;
    if ((st = setup_fft(ctx, (size_t)batch * H * (W / 2 + 1)))) return st;
    if ((st = dalloc(ctx, &p, sizeof(float) * H * (W / 2 + 1)))) return st;
    ctx->mhalf = (float*)p;
    if ((st = dalloc(ctx, &p, sizeof(float) * H * (W / 2 + 1)))) return st;
    ctx->dgl = (float*)p;
  } else if (op->kind == IDEQ_OP_RICIAN) {
    if (op->step == IDEQ_STEP_PROX) return fail(ctx, IDEQ_E_UNSUPPORTED, "no closed-form Rician prox (PAPER l.1079)");
    if (!(op->sigma > 0.f)) return fail(ctx, IDEQ_E_INVALID, "Rician sigma must be > 0");
  } else {
    return fail(ctx, IDEQ_E_INVALID, "unknown operator kind");
  }
  ctx->op = *op;
  ctx->op.kernels = nullptr;
  ctx->op.masks = nullptr;
  ctx->op.phase_masks = nullptr;
  ctx->op_batch = batch;
  ctx->op_set = true;
  ctx->graph_key.clear();
  return IDEQ_OK;
}

ideq_status ideq_solve(ideq_ctx* ctx, const float* y, float* x_inout, int batch, const ideq_params* p,
                       ideq_image_stat* stats, float* rmax_trace) {
  ideq_status st;
  if ((st = check_ctx(ctx))) return st;
  return solve_device(ctx, y, x_inout, batch, p, stats, rmax_trace);
}

ideq_status ideq_solve_host(ideq_ctx* ctx, const float* y, float* x_inout, int batch, const ideq_params* p,
                            ideq_image_stat* stats, float* rmax_trace) {
  ideq_status st;
  if ((st = check_ctx(ctx))) return st;
  if (!y || !x_inout) return fail(ctx, IDEQ_E_INVALID, "NULL y/x");
  if (batch < 1 || batch > ctx->maxN) return fail(ctx, IDEQ_E_INVALID, "batch out of range");
  const size_t cy = !ctx->op_set ? (size_t)ctx->C
                    : ctx->op.kind == IDEQ_OP_PHASE ? (size_t)ctx->op.n_phase
                    : ctx->op.kind == IDEQ_OP_MRI ? (size_t)2 : (size_t)ctx->C;  // MRI: complex k-space
  const size_t ny = (size_t)batch * cy * ctx->H * ctx->W, nx = (size_t)batch * ctx->C * ctx->H * ctx->W;
  if (ny > ctx->dstage_y_n) {
    void* p2;
    if ((st = dalloc(ctx, &p2, ny * 4))) return st;
    ctx->dstage_y = (float*)p2;
    ctx->dstage_y_n = ny;
    ctx->graph_key.clear();
  }
  if (nx > ctx->dstage_x_n) {
    void* p2;
    if ((st = dalloc(ctx, &p2, nx * 4))) return st;
    ctx->dstage_x = (float*)p2;
    ctx->dstage_x_n = nx;
    ctx->graph_key.clear();
  }
  CK(cudaMemcpyAsync(ctx->dstage_y, y, ny * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->dstage_x, x_inout, nx * 4, cudaMemcpyHostToDevice, ctx->stream));
  st = solve_device(ctx, ctx->dstage_y, ctx->dstage_x, batch, p, stats, rmax_trace);
  if (st != IDEQ_OK && st != IDEQ_E_DIVERGED) return st;
  CK(cudaMemcpyAsync(x_inout, ctx->dstage_x, nx * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return st;
}

ideq_status ideq_grad_g(ideq_ctx* ctx, const float* z, float* grad_out, float* u_out, int batch) {
  ideq_status st;
  if ((st = check_ctx(ctx))) return st;
  if (!z || !grad_out) return fail(ctx, IDEQ_E_INVALID, "NULL z/grad");
  if (batch < 1 || batch > ctx->maxN) return fail(ctx, IDEQ_E_INVALID, "batch out of range");
  if ((st = prepare_programs(ctx, batch))) return st;
  const size_t n = (size_t)batch * ctx->C * ctx->H * ctx->W;
  CK(cudaMemcpyAsync(ctx->Z, z, n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  launch_init_state(make_fin(ctx, batch, nullptr), ctx->stream);  // every image active: no tile skipped
  ctx->skip_frozen = false;
  enable_skip(ctx, false);
  run_network(ctx, batch);
  CK(cudaMemcpyAsync(grad_out, ctx->G, n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  if (u_out) CK(cudaMemcpyAsync(u_out, ctx->Hc, n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaGetLastError());
  collect_profile(ctx);
  return IDEQ_OK;
}

ideq_status ideq_fidelity_grad(ideq_ctx* ctx, const float* y, const float* x, float* out, int batch) {
  ideq_status st;
  if ((st = check_ctx(ctx))) return st;
  if (!ctx->op_set) return fail(ctx, IDEQ_E_STATE, "no operator");
  if (!y || !x || !out || batch < 1 || batch > ctx->op_batch) return fail(ctx, IDEQ_E_INVALID, "bad arguments");
  const auto& op = ctx->op;
  if (op.kind == IDEQ_OP_INPAINT) {
    launch_inpaint_grad(x, y, ctx->d_mask, out, batch, ctx->C, ctx->H, ctx->W, ctx->stream);
  } else if (op.kind == IDEQ_OP_MRI) {
    prepare_mri(ctx, y, 1.f, batch);
    FftArgs f = make_fft_args(ctx, y, nullptr);
    f.dgl = ctx->mhalf;
    f.active = nullptr;
    StepArgs dummy{};
    launch_blur_rows_fwd(f, x, 0, batch, ctx->stream);
    launch_blur_cols(f, 0, batch, ctx->stream);
    launch_blur_rows_inv(f, dummy, ctx->fbuf, 0, batch, ctx->stream);
    launch_sub(ctx->fbuf, ctx->fbuf2, out, (long long)batch * ctx->H * ctx->W, ctx->stream);
  } else if (op.kind == IDEQ_OP_RICIAN) {
    launch_rician_grad(x, y, 1.f / (op.sigma * op.sigma), out, (long long)batch * ctx->C * ctx->H * ctx->W,
                       ctx->stream);
  } else if (op.kind == IDEQ_OP_BLUR && op.blur_impl == IDEQ_BLUR_DIRECT) {
    StepArgs a = make_step_args(ctx, batch, y, nullptr, nullptr);
    a.z = x;
    a.active = nullptr;
    a.fbuf2 = out;
    launch_blur_residual(a, ctx->stream);
    launch_blur_adjoint(0, a, ctx->fbuf, ctx->stream);
  } else if (op.kind == IDEQ_OP_PHASE) {
    FftArgs f = make_fft_args(ctx, y, nullptr);
    f.z = x;
    f.active = nullptr;
    StepArgs dummy{};
    launch_phase_rows_fwd(f, batch, ctx->stream);
    launch_phase_cols(f, batch, ctx->stream);
    launch_phase_rows_inv(f, dummy, out, 0, batch, ctx->stream);
  } else {
    return fail(ctx, IDEQ_E_UNSUPPORTED, "the blur gradient uses blur_impl DIRECT");
  }
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaGetLastError());
  return IDEQ_OK;
}

ideq_status ideq_fidelity_prox(ideq_ctx* ctx, const float* y, const float* v, float tau, float* out, int batch) {
  ideq_status st;
  if ((st = check_ctx(ctx))) return st;
  if (!ctx->op_set) return fail(ctx, IDEQ_E_STATE, "no operator");
  if (!y || !v || !out || batch < 1 || batch > ctx->op_batch || !(tau > 0.f)) return fail(ctx, IDEQ_E_INVALID, "bad arguments");
  if (ctx->op.kind == IDEQ_OP_INPAINT) {
    launch_inpaint_prox(v, y, ctx->d_mask, tau, out, batch, ctx->C, ctx->H, ctx->W, ctx->stream);
  } else if (ctx->op.kind == IDEQ_OP_MRI) {
    prepare_mri(ctx, y, tau, batch);
    FftArgs f = make_fft_args(ctx, y, nullptr);
    f.z = v; f.gg = v; f.lam = 0.f; f.tau = tau;
    f.active = nullptr;
    StepArgs dummy{};
    launch_blur_rows_fwd(f, nullptr, 1, batch, ctx->stream);
    launch_blur_cols(f, 0, batch, ctx->stream);
    launch_blur_rows_inv(f, dummy, out, 0, batch, ctx->stream);
  } else if (ctx->op.kind == IDEQ_OP_PHASE || ctx->op.kind == IDEQ_OP_RICIAN) {
    return fail(ctx, IDEQ_E_UNSUPPORTED, "no closed-form prox for phase retrieval / Rician (PAPER l.1079)");
  } else if (ctx->op.blur_impl == IDEQ_BLUR_FFT) {
    // prox_{tau f}(v) = F^-1[F(v + tau A^T y) / (1 + tau |K^|^2)]: the solver's passes with lam = 0
    prepare_blur_prox(ctx, y, tau, batch);
    FftArgs f = make_fft_args(ctx, y, nullptr);
    f.z = v; f.gg = v; f.lam = 0.f; f.tau = tau;
    f.active = nullptr;
    StepArgs dummy{};
    launch_blur_rows_fwd(f, nullptr, 1, batch, ctx->stream);
    launch_blur_cols(f, 0, batch, ctx->stream);
    launch_blur_rows_inv(f, dummy, out, 0, batch, ctx->stream);
  } else {
    return fail(ctx, IDEQ_E_UNSUPPORTED, "the blur prox needs blur_impl FFT");
  }
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaGetLastError());
  return IDEQ_OK;
}

// ======================================================================== JFB gradient (NEXT-4)
// dL/dtheta, dL/dlam, dL/dtau of L = 1/2 sum_i ||T(x_hat_i) - x*_i||^2 with one more i-DEQ step at
// the fixed point (z = x_hat, so dL/dbeta = 0); see jfb.cu and oracle/jfb.py. fp32 FFMA path.
namespace {

struct JfbRun {
  ideq_ctx* ctx;
  int N;
  cudaStream_t s;
  std::map<std::string, float*> dw;  // per weight tensor: gradient in the layer's operand / blob layout
  WeightSlices ws;
  ideq_status st = IDEQ_OK;

  size_t nbuf = 0;  // tape blocks handed out by this call (index into ctx->jfb_pool)
  float* work(size_t n) {
    if (n > ctx->jfb_ws_n) {
      if (ctx->jfb_ws) { cudaStreamSynchronize(s); cudaFree(ctx->jfb_ws); ctx->jfb_ws = nullptr; ctx->jfb_ws_n = 0; }
      if (cudaMalloc(&ctx->jfb_ws, n * sizeof(float)) != cudaSuccess) {
        cudaGetLastError(); ctx->jfb_ws = nullptr; st = IDEQ_E_NOMEM; return nullptr;
      }
      ctx->jfb_ws_n = n;
    }
    return ctx->jfb_ws;
  }
  // zeroed device block; the i-th request of a call reuses the i-th block of the previous call
  // when it is large enough (the request sequence depends only on the shapes)
  float* buf(size_t n) {
    const size_t bytes = (n ? n : 1) * sizeof(float);
    auto& pool = ctx->jfb_pool;
    if (nbuf == pool.size()) pool.push_back({nullptr, 0});
    auto& b = pool[nbuf++];
    if (b.second < bytes) {
      if (b.first) { cudaStreamSynchronize(s); cudaFree(b.first); b = {nullptr, 0}; }
      if (cudaMalloc(&b.first, bytes) != cudaSuccess) { cudaGetLastError(); st = IDEQ_E_NOMEM; return nullptr; }
      b.second = bytes;
    }
    cudaMemsetAsync(b.first, 0, bytes, s);
    return (float*)b.first;
  }

  // shape-derived GEMM quantities of a layer, as in add_gemm_w
  void dims(int kind, const std::vector<int>& shp, int& ncols, int& ktap, int& cin) {
    if (kind == 0) { ncols = shp[0]; ktap = shp[1]; }
    else if (kind == 1) { ncols = shp[1]; ktap = shp[0]; }
    else if (kind == 2 || kind == 5) { ncols = shp[0]; ktap = 2 * shp[1]; }
    else { ncols = 4 * shp[1]; ktap = shp[0]; }
    cin = (kind == 2 || kind == 5) ? ktap / 2 : ktap;
  }
  const float* weights(const std::string& wname, int kind, int KC) {
    const std::string key = wname + "#" + std::to_string(kind) + "simt";
    if (!ctx->wdev.count(key)) {
      auto& sl = ws.t[wname];
      int ncols, ntaps, ktap;
      std::vector<float> B = gemm_weights(kind, ctx->blob.data() + sl.first, sl.second, KC, ncols, ntaps, ktap);
      if (upload_gemm_weights(ctx, key, B)) { st = IDEQ_E_CUDA; return nullptr; }
    }
    return (const float*)ctx->wdev[key];
  }
  ConvGeom geom(const std::string& wname, int kind, int Hin, int Win, int epi) {
    int ncols, ktap, cin;
    dims(kind, ws.t[wname].second, ncols, ktap, cin);
    return make_geom(kind, N, Hin, Win, cin, ncols, pick_kc(false, ktap), ktap, epi);
  }
  // One layer of the two-stream passes. With the tensor-core fp32 mode (3xTF32) the layer runs on
  // the solver's own tcgen05 kernel (same GEMM operands, hi / lo tf32 halves); the plan binds the
  // tape buffers, which keep their addresses across calls (the pool hands out the same blocks), so
  // it is built once per (layer, buffers). Otherwise the FFMA implicit GEMM.
  void conv(const std::string& wname, int kind, int Hin, int Win, const float* in, float* out, const float* aux,
            int epi) {
    if (use_x3(ctx)) {
      char key[256];
      snprintf(key, sizeof(key), "%s#%d#%d#%d#%d#%d#%p#%p#%p", wname.c_str(), kind, N, Hin, Win, epi, (const void*)in,
               (const void*)out, (const void*)aux);
      auto it = ctx->jfb_plans.find(key);
      if (it == ctx->jfb_plans.end()) {
        int ncols, ktap, cin;
        dims(kind, ws.t[wname].second, ncols, ktap, cin);
        const ConvGeom g = make_geom(kind, N, Hin, Win, cin, ncols, pick_kc(true, true, ktap), ktap, epi);
        TcPlan* plan = nullptr;
        if (tc_supported(g, true)) {
          const std::string wk = wname + "#" + std::to_string(kind) + "x3";
          if (!ctx->wdev.count(wk)) {  // hi / lo tf32 halves of the GEMM operand
            auto& sl = ws.t[wname];
            int nc, nt, kt;
            std::vector<float> B = gemm_weights(kind, ctx->blob.data() + sl.first, sl.second, g.KC, nc, nt, kt);
            std::vector<float> lo(B.size());
            for (size_t i = 0; i < B.size(); ++i) {
              const float h = tf32_rna(B[i]);
              lo[i] = tf32_rna(B[i] - h);
              B[i] = h;
            }
            if (upload_gemm_weights(ctx, wk + "#lo", lo) || upload_gemm_weights(ctx, wk, B)) { st = IDEQ_E_CUDA; return; }
          }
          char err[256] = {0};
          plan = tc_make_plan(g, true, in, ctx->wdev[wk], ctx->wdev[wk + "#lo"], out, aux, ctx->num_sms, err, sizeof(err));
        }
        it = ctx->jfb_plans.emplace(key, plan).first;  // null: geometry the tensor-core path does not take
      }
      if (it->second) {
        tc_launch(it->second, s);
        return;
      }
    }
    ConvGeom g = geom(wname, kind, Hin, Win, epi);
    const float* w = weights(wname, kind, g.KC);
    if (w) launch_conv_simt<float>(g, in, w, out, aux, s);
  }
  // weight gradient of the FORWARD layer (kind 0 / 2 / 4) for one stream, accumulated
  void wgrad(const std::string& wname, int kind, int Hin, int Win, const float* in, const float* gout) {
    ConvGeom g = geom(wname, kind, Hin, Win, EPI_STORE);
    float*& d = dw[wname];
    if (!d) d = buf((size_t)g.ntaps * g.nchunk * g.ncols * g.KC);
    float* w = work(wgrad_workspace(g));
    if (d && w) launch_wgrad_geom(g, in, gout, d, w, s);
  }
  const float* headtail_w(const std::string& wname, bool adjoint) {
    const std::string key = wname + (adjoint ? "#T" : "#F");
    if (!ctx->wdev.count(key)) {
      auto& sl = ws.t[wname];
      const float* Wt = ctx->blob.data() + sl.first;
      std::vector<float> v;
      if (adjoint) v = flip_transpose3x3(Wt, sl.second[0], sl.second[1]);
      else v.assign(Wt, Wt + (size_t)sl.second[0] * sl.second[1] * 9);
      if (upload_f32(ctx, key, v)) { st = IDEQ_E_CUDA; return nullptr; }
    }
    return (const float*)ctx->wdev[key];
  }
  void head_wgrad(const std::string& wname, const float* img, const float* gf, int C, int H, int W, int wf) {
    float* d = dw_blob(wname);
    float* w = work(headtail_wgrad_workspace(N, C, H, wf));
    if (d && w) launch_head_wgrad(img, gf, d, w, N, C, H, W, wf, s);
  }
  void tail_wgrad(const std::string& wname, const float* f, const float* gimg, int C, int H, int W, int wf) {
    float* d = dw_blob(wname);
    float* w = work(headtail_wgrad_workspace(N, C, H, wf));
    if (d && w) launch_tail_wgrad(f, gimg, d, w, N, C, H, W, wf, s);
  }
  float* dw_blob(const std::string& wname) {  // head / tail: gradient directly in blob layout
    float*& d = dw[wname];
    if (!d) {
      auto& shp = ws.t[wname].second;
      d = buf((size_t)shp[0] * shp[1] * shp[2] * shp[3]);
    }
    return d;
  }
};

}  // namespace

ideq_status ideq_jfb_grad(ideq_ctx* ctx, const float* y, const float* x_hat, const float* x_star, int batch,
                          const ideq_params* p, float* dtheta, float* dlam, float* dtau, float* dbeta, float* loss) {
  ideq_status st;
  if ((st = check_ctx(ctx))) return st;
  if (!y || !x_hat || !x_star || !p || !dtheta || !dlam || !dtau || !dbeta || !loss)
    return fail(ctx, IDEQ_E_INVALID, "NULL argument");
  if (batch < 1 || batch > ctx->maxN) return fail(ctx, IDEQ_E_INVALID, "batch out of range");
  if (ctx->prec != IDEQ_PREC_FP32) return fail(ctx, IDEQ_E_UNSUPPORTED, "the JFB gradient runs in the fp32 mode");
  if (!ctx->net.identity_skip) return fail(ctx, IDEQ_E_UNSUPPORTED, "the JFB gradient assumes N = z + U");
  if (ctx->net.act != IDEQ_ACT_SOFTPLUS) return fail(ctx, IDEQ_E_UNSUPPORTED, "the JFB gradient assumes softplus");
  if (!ctx->op_set) return fail(ctx, IDEQ_E_STATE, "no operator");
  const bool prox = ctx->op.step == IDEQ_STEP_PROX;
  if (prox && ctx->op.kind != IDEQ_OP_INPAINT)
    return fail(ctx, IDEQ_E_UNSUPPORTED, "JFB prox variant: inpainting (closed-form Jacobian) only");
  const int C = ctx->C, H = ctx->H, W = ctx->W;
  const long long nimg = (long long)batch * C * H * W;
  JfbRun J;
  J.ctx = ctx;
  J.N = batch;
  J.s = ctx->stream;
  size_t tot;
  slice_weights(ctx->net, J.ws, tot);
  cudaStream_t s = ctx->stream;
  // ---- grad g(z), U(z) at z = x_hat; grad f(z) (gradient variant)
  float* gg = J.buf(nimg);
  float* U = J.buf(nimg);
  float* gf = J.buf(nimg);
  float* v = J.buf(nimg);
  float* terms = J.buf(3 * nimg);
  double* dsum = (double*)J.buf(8);          // 4 doubles
  double* dpart = (double*)J.buf(2 * 3 * 256);  // 3 x 256 doubles
  if (J.st) return fail(ctx, IDEQ_E_NOMEM, "JFB workspace");
  if ((st = ideq_grad_g(ctx, x_hat, gg, U, batch))) return st;
  if (!prox && (st = ideq_fidelity_grad(ctx, y, x_hat, gf, batch))) return st;
  launch_jfb_residual(x_hat, x_star, gg, gf, y, ctx->d_mask, prox ? 1 : 0, p->lambda, p->tau, nimg, (long long)H * W,
                      (long long)C * H * W, v, terms, s);
  launch_sums(terms, nimg, 3, dpart, dsum, s);
  // ---- two-stream forward (primal z, tangent v) with a tape, reverse with weight gradients
  const auto& n = ctx->net;
  const long long HW = (long long)H * W;
  if (n.arch == IDEQ_NET_TINY3) {
    const int w = n.widths[0];
    const long long nf = (long long)batch * HW * w;
    float *p1 = J.buf(nf), *a1 = J.buf(nf), *p1d = J.buf(nf), *a1d = J.buf(nf);
    float *p2 = J.buf(nf), *a2 = J.buf(nf), *p2d = J.buf(nf), *a2d = J.buf(nf);
    float *Ud = J.buf(nimg), *Up = J.buf(nimg);
    if (J.st) return fail(ctx, J.st, "JFB workspace");
    launch_img2feat<float>(x_hat, J.headtail_w("c1", false), p1, nullptr, EPI_STORE, batch, C, H, W, w, s);
    launch_img2feat<float>(v, J.headtail_w("c1", false), p1d, nullptr, EPI_STORE, batch, C, H, W, w, s);
    launch_sp_forward(p1, a1, nf, s);
    launch_sp_tangent(a1, p1d, a1d, nf, s);
    J.conv("c2", 0, H, W, a1, p2, nullptr, EPI_STORE);
    J.conv("c2", 0, H, W, a1d, p2d, nullptr, EPI_STORE);
    launch_sp_forward(p2, a2, nf, s);
    launch_sp_tangent(a2, p2d, a2d, nf, s);
    launch_feat2img<float>(a2, J.headtail_w("c3", false), Up, nullptr, 0.f, batch, C, H, W, w, s);
    launch_feat2img<float>(a2d, J.headtail_w("c3", false), Ud, nullptr, 0.f, batch, C, H, W, w, s);
    // reverse: U_bar = U_dot, U_dot_bar = U
    J.tail_wgrad("c3", a2, Ud, C, H, W, w);
    J.tail_wgrad("c3", a2d, Up, C, H, W, w);
    float *a2b = J.buf(nf), *a2db = J.buf(nf), *p2b = J.buf(nf), *p2db = J.buf(nf);
    float *a1b = J.buf(nf), *a1db = J.buf(nf), *p1b = J.buf(nf), *p1db = J.buf(nf);
    if (J.st) return fail(ctx, J.st, "JFB workspace");
    launch_img2feat<float>(Ud, J.headtail_w("c3", true), a2b, nullptr, EPI_STORE, batch, C, H, W, w, s);
    launch_img2feat<float>(Up, J.headtail_w("c3", true), a2db, nullptr, EPI_STORE, batch, C, H, W, w, s);
    launch_sp_reverse(a2, p2d, a2b, a2db, p2b, p2db, nf, s);
    J.wgrad("c2", 0, H, W, a1, p2b);
    J.wgrad("c2", 0, H, W, a1d, p2db);
    J.conv("c2", 1, H, W, p2b, a1b, nullptr, EPI_STORE);
    J.conv("c2", 1, H, W, p2db, a1db, nullptr, EPI_STORE);
    launch_sp_reverse(a1, p1d, a1b, a1db, p1b, p1db, nf, s);
    J.head_wgrad("c1", x_hat, p1b, C, H, W, w);
    J.head_wgrad("c1", v, p1db, C, H, W, w);
  } else {
    const int R = n.res_blocks;
    int Hl[4], Wl[4], wl[4];
    for (int l = 0; l < 4; ++l) { Hl[l] = H >> l; Wl[l] = W >> l; wl[l] = n.widths[l]; }
    auto fsz = [&](int l) { return (long long)batch * Hl[l] * Wl[l] * wl[l]; };
    struct Rec { int kind, l; std::string nA, nB; const float *x, *xd; float *a, *pd, *ad; };
    std::vector<Rec> tape;
    float* t = J.buf(fsz(0));
    float* td = J.buf(fsz(0));
    if (J.st) return fail(ctx, J.st, "JFB workspace");
    launch_img2feat<float>(x_hat, J.headtail_w("head", false), t, nullptr, EPI_STORE, batch, C, H, W, wl[0], s);
    launch_img2feat<float>(v, J.headtail_w("head", false), td, nullptr, EPI_STORE, batch, C, H, W, wl[0], s);
    const float* skip[3] = {nullptr, nullptr, nullptr};
    const float* skipd[3] = {nullptr, nullptr, nullptr};
    auto rb_fwd = [&](const char* pre, int l, int r) {
      const std::string nA = std::string(pre) + std::to_string(l) + "." + std::to_string(r) + ".A";
      const std::string nB = std::string(pre) + std::to_string(l) + "." + std::to_string(r) + ".B";
      const long long nf = fsz(l);
      float *pp = J.buf(nf), *a = J.buf(nf), *pd = J.buf(nf), *ad = J.buf(nf), *t2 = J.buf(nf), *t2d = J.buf(nf);
      if (J.st) return;
      J.conv(nA, 0, Hl[l], Wl[l], t, pp, nullptr, EPI_STORE);
      launch_sp_forward(pp, a, nf, s);
      J.conv(nA, 0, Hl[l], Wl[l], td, pd, nullptr, EPI_STORE);
      launch_sp_tangent(a, pd, ad, nf, s);
      J.conv(nB, 0, Hl[l], Wl[l], a, t2, t, EPI_RESADD);
      J.conv(nB, 0, Hl[l], Wl[l], ad, t2d, td, EPI_RESADD);
      tape.push_back({0, l, nA, nB, t, td, a, pd, ad});
      t = t2;
      td = t2d;
    };
    for (int l = 0; l < 4; ++l) {
      for (int r = 0; r < R; ++r) rb_fwd("e", l, r);
      if (l < 3) {
        skip[l] = t;
        skipd[l] = td;
        tape.push_back({1, l, "down" + std::to_string(l), "", t, td, nullptr, nullptr, nullptr});
        float *c = J.buf(fsz(l + 1)), *cd = J.buf(fsz(l + 1));
        if (J.st) return fail(ctx, J.st, "JFB workspace");
        J.conv("down" + std::to_string(l), 2, Hl[l], Wl[l], t, c, nullptr, EPI_STORE);
        J.conv("down" + std::to_string(l), 2, Hl[l], Wl[l], td, cd, nullptr, EPI_STORE);
        t = c;
        td = cd;
      }
    }
    for (int l = 2; l >= 0; --l) {
      tape.push_back({2, l, "up" + std::to_string(l), "", t, td, nullptr, nullptr, nullptr});
      float *f = J.buf(fsz(l)), *fd = J.buf(fsz(l));
      if (J.st) return fail(ctx, J.st, "JFB workspace");
      J.conv("up" + std::to_string(l), 4, Hl[l + 1], Wl[l + 1], t, f, skip[l], EPI_RESADD);
      J.conv("up" + std::to_string(l), 4, Hl[l + 1], Wl[l + 1], td, fd, skipd[l], EPI_RESADD);
      t = f;
      td = fd;
      for (int r = 0; r < R; ++r) rb_fwd("d", l, r);
    }
    if (J.st) return fail(ctx, J.st, "JFB workspace");
    float *Up = J.buf(nimg), *Ud = J.buf(nimg);
    float *gb = J.buf(fsz(0)), *gdb = J.buf(fsz(0));
    if (J.st) return fail(ctx, J.st, "JFB workspace");
    launch_feat2img<float>(t, J.headtail_w("tail", false), Up, nullptr, 0.f, batch, C, H, W, wl[0], s);
    launch_feat2img<float>(td, J.headtail_w("tail", false), Ud, nullptr, 0.f, batch, C, H, W, wl[0], s);
    // reverse: U_bar = U_dot, U_dot_bar = U
    J.tail_wgrad("tail", t, Ud, C, H, W, wl[0]);
    J.tail_wgrad("tail", td, Up, C, H, W, wl[0]);
    launch_img2feat<float>(Ud, J.headtail_w("tail", true), gb, nullptr, EPI_STORE, batch, C, H, W, wl[0], s);
    launch_img2feat<float>(Up, J.headtail_w("tail", true), gdb, nullptr, EPI_STORE, batch, C, H, W, wl[0], s);
    const float* sb[3] = {nullptr, nullptr, nullptr};
    const float* sdb[3] = {nullptr, nullptr, nullptr};
    for (int i = (int)tape.size() - 1; i >= 0; --i) {
      const Rec& rc = tape[i];
      const int l = rc.l;
      const long long nf = fsz(l);
      if (rc.kind == 0) {  // t' = t + B(sp(A t))
        float *ab = J.buf(nf), *adb = J.buf(nf), *pb = J.buf(nf), *pdb = J.buf(nf), *g2 = J.buf(nf), *g2d = J.buf(nf);
        if (J.st) return fail(ctx, J.st, "JFB workspace");
        J.conv(rc.nB, 1, Hl[l], Wl[l], gb, ab, nullptr, EPI_STORE);
        J.conv(rc.nB, 1, Hl[l], Wl[l], gdb, adb, nullptr, EPI_STORE);
        J.wgrad(rc.nB, 0, Hl[l], Wl[l], rc.a, gb);
        J.wgrad(rc.nB, 0, Hl[l], Wl[l], rc.ad, gdb);
        launch_sp_reverse(rc.a, rc.pd, ab, adb, pb, pdb, nf, s);
        J.wgrad(rc.nA, 0, Hl[l], Wl[l], rc.x, pb);
        J.wgrad(rc.nA, 0, Hl[l], Wl[l], rc.xd, pdb);
        J.conv(rc.nA, 1, Hl[l], Wl[l], pb, g2, gb, EPI_RESADD);
        J.conv(rc.nA, 1, Hl[l], Wl[l], pdb, g2d, gdb, EPI_RESADD);
        gb = g2;
        gdb = g2d;
      } else if (rc.kind == 2) {  // t = up(x) + s_l: the skip's cotangent is t's
        sb[l] = gb;
        sdb[l] = gdb;
        float *c = J.buf(fsz(l + 1)), *cd = J.buf(fsz(l + 1));
        if (J.st) return fail(ctx, J.st, "JFB workspace");
        J.wgrad(rc.nA, 4, Hl[l + 1], Wl[l + 1], rc.x, gb);
        J.wgrad(rc.nA, 4, Hl[l + 1], Wl[l + 1], rc.xd, gdb);
        J.conv(rc.nA, 5, Hl[l], Wl[l], gb, c, nullptr, EPI_STORE);
        J.conv(rc.nA, 5, Hl[l], Wl[l], gdb, cd, nullptr, EPI_STORE);
        gb = c;
        gdb = cd;
      } else {  // x -> down(x), and x = s_l
        float *f = J.buf(nf), *fd = J.buf(nf);
        if (J.st) return fail(ctx, J.st, "JFB workspace");
        J.wgrad(rc.nA, 2, Hl[l], Wl[l], rc.x, gb);
        J.wgrad(rc.nA, 2, Hl[l], Wl[l], rc.xd, gdb);
        J.conv(rc.nA, 3, Hl[l + 1], Wl[l + 1], gb, f, sb[l], EPI_RESADD);
        J.conv(rc.nA, 3, Hl[l + 1], Wl[l + 1], gdb, fd, sdb[l], EPI_RESADD);
        gb = f;
        gdb = fd;
      }
    }
    J.head_wgrad("head", x_hat, gb, C, H, W, wl[0]);
    J.head_wgrad("head", v, gdb, C, H, W, wl[0]);
  }
  if (J.st) return fail(ctx, J.st, "JFB workspace / weights");
  // ---- scale by -tau lam, bring back, map each layer operand layout to the blob order
  const float scale = -p->tau * p->lambda;
  std::vector<float> host;
  for (auto& kv : J.dw) {
    const std::string& name = kv.first;
    auto& sl = J.ws.t[name];
    const std::vector<int>& shp = sl.second;
    const size_t nw = (size_t)shp[0] * shp[1] * shp[2] * shp[3];
    const bool headtail = (name == "head" || name == "tail" || name == "c1" || name == "c3");
    if (headtail) {
      launch_scale(kv.second, scale, (long long)nw, s);
      CK(cudaMemcpyAsync(dtheta + sl.first, kv.second, nw * sizeof(float), cudaMemcpyDeviceToHost, s));
      continue;
    }
    const int kind = name.compare(0, 4, "down") == 0 ? 2 : name.compare(0, 2, "up") == 0 ? 4 : 0;
    int ncols, ktap, cin;
    J.dims(kind, shp, ncols, ktap, cin);
    const int KC = pick_kc(false, ktap);
    // operand index -> blob index: gemm_weights applied to the blob positions themselves (cached)
    std::vector<uint32_t>& map = ctx->jfb_map[name];
    if (map.empty()) {
      std::vector<float> pos(nw);
      for (size_t i = 0; i < nw; ++i) pos[i] = (float)i;  // exact: nw < 2^24
      int nc2, nt2, kt2;
      std::vector<float> m = gemm_weights(kind, pos.data(), shp, KC, nc2, nt2, kt2);
      map.assign(m.begin(), m.end());
    }
    const size_t nb = map.size();
    launch_scale(kv.second, scale, (long long)nb, s);
    host.resize(nb);
    CK(cudaMemcpyAsync(host.data(), kv.second, nb * sizeof(float), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (size_t b = 0; b < nb; ++b) dtheta[sl.first + (size_t)map[b]] = host[b];  // permutation only
  }
  double sums[3];
  CK(cudaMemcpyAsync(sums, dsum, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  *loss = (float)sums[0];
  *dlam = (float)sums[1];
  *dtau = (float)sums[2];
  *dbeta = 0.f;  // z = x_hat + beta (x_hat - x_hat)
  return IDEQ_OK;
}

ideq_status ideq_time_class(ideq_ctx* ctx, int cls, int reps, double* ms, double* flops, double* bytes,
                            double* iter_ms) {
  ideq_status st;
  if ((st = check_ctx(ctx))) return st;
  if (!ctx->have_last) return fail(ctx, IDEQ_E_STATE, "ideq_time_class needs a solve first");
  if (ctx->last_fused)
    return fail(ctx, IDEQ_E_UNSUPPORTED, "the last solve ran the whole-solve kernel: no iteration graph to time");
  if (!ms || reps < 1 || cls < 0 || cls >= IDEQ_K_NCLASSES || cls == IDEQ_K_FIDELITY)
    return fail(ctx, IDEQ_E_INVALID, "class must be CONV_TC, CONV_SIMT, HEADTAIL, STEP or REDUCE; reps >= 1");
  cudaStream_t s = ctx->stream;
  // one whole iteration of the last solve (same kernels, order and launch configuration as its
  // graph) with event-record nodes at the class boundaries; the update writes x^{k+1} into
  // scratch, never into the caller's x (the context's solver state is overwritten)
  StepArgs a = ctx->last_a;
  a.X0 = ctx->Xsnap;
  FinalizeArgs f = ctx->last_f;
  f.trace = nullptr;
  SegTimer T;
  T.s = s;
  const bool prof = ctx->profiling;
  ctx->profiling = false;
  ctx->counting = true;
  for (int k = 0; k < IDEQ_K_NCLASSES; ++k) ctx->cnt_flops[k] = ctx->cnt_bytes[k] = 0.0;
  cudaGraph_t graph;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  ctx->segt = &T;
  ideq_status st2 = enqueue_iteration(ctx, a, f, false);
  T.close();
  ctx->segt = nullptr;
  cudaError_t ec = cudaStreamEndCapture(s, &graph);
  ctx->counting = false;
  ctx->profiling = prof;
  if (st2) return st2;
  if (ec != cudaSuccess) return fail(ctx, IDEQ_E_CUDA, "class capture: %s", cudaGetErrorString(ec));
  cudaGraphExec_t ge;
  CK(cudaGraphInstantiate(&ge, graph, 0));
  cudaGraphDestroy(graph);
  CK(cudaGraphLaunch(ge, s));  // warm-up
  CK(cudaStreamSynchronize(s));
  double tot = 0.0, all = 0.0;
  for (int r = 0; r < reps; ++r) {
    CK(cudaGraphLaunch(ge, s));
    CK(cudaStreamSynchronize(s));
    for (int c = 0; c < IDEQ_K_NCLASSES; ++c)
      for (auto& pr : T.seg[c]) {
        float t = 0.f;
        cudaError_t e = cudaEventElapsedTime(&t, pr.first, pr.second);
        if (e != cudaSuccess) { cudaGraphExecDestroy(ge); return fail(ctx, IDEQ_E_CUDA, "class timing: %s", cudaGetErrorString(e)); }
        all += t;
        if (c == cls) tot += t;
      }
  }
  cudaGraphExecDestroy(ge);
  *ms = tot / reps;
  if (iter_ms) *iter_ms = all / reps;
  const bool step = cls == IDEQ_K_STEP;  // the step's fidelity passes count with it
  if (flops) *flops = ctx->cnt_flops[cls] + (step ? ctx->cnt_flops[IDEQ_K_FIDELITY] : 0.0);
  if (bytes) *bytes = ctx->cnt_bytes[cls] + (step ? ctx->cnt_bytes[IDEQ_K_FIDELITY] : 0.0);
  return IDEQ_OK;
}

ideq_status ideq_set_profiling(ideq_ctx* ctx, int enable) {
  if (!ctx) return IDEQ_E_INVALID;
  ctx->profiling = enable != 0;
  return IDEQ_OK;
}

ideq_status ideq_get_profile(ideq_ctx* ctx, ideq_profile* out, int reset) {
  if (!ctx || !out) return IDEQ_E_INVALID;
  collect_profile(ctx);
  *out = ctx->prof;
  if (reset) memset(&ctx->prof, 0, sizeof(ctx->prof));
  return IDEQ_OK;
}

int ideq_launches_per_iteration(const ideq_ctx* ctx) {
  if (!ctx || !ctx->have_last || ctx->last_fused) return 0;  // fused: one launch per solve
  int n = 0;
  for (int first = 0; first < ctx->last_N; first += ctx->mb) {
    const int m = ctx->last_N - first < ctx->mb ? ctx->last_N - first : ctx->mb;
    auto it = ctx->progs.find(m);
    if (it != ctx->progs.end()) n += (int)it->second.layers.size();
  }
  if (ctx->op.kind == IDEQ_OP_BLUR) n += 2; else n += 1;
  n += 3;  // finalize, advance_a, advance_b
  return n;
}

int ideq_debug_conv(int kind, int precision, int use_tc_, const float* w, int s0, int s1, int N, int Hin, int Win,
                    const void* in, void* out, const void* aux, int epi, char* err, int errlen) {
  auto seterr = [&](const char* m) { if (err && errlen > 0) { snprintf(err, errlen, "%s", m); } };
  if (kind < 0 || kind > 5 || !w || !in || !out) { seterr("bad arguments"); return IDEQ_E_INVALID; }
  init_kernel_attributes();
  const bool x3 = use_tc_ && precision == IDEQ_PREC_FP32;  // fp32 on tcgen05 = 3xTF32
  const int kh = (kind <= 1) ? 3 : 2;
  std::vector<int> shp = {s0, s1, kh, kh};
  int ncols = 0, ntaps = 0, ktap = 0;
  if (kind == 0) { ncols = s0; ktap = s1; }
  else if (kind == 1) { ncols = s1; ktap = s0; }
  else if (kind == 2 || kind == 5) { ncols = s0; ktap = 2 * s1; }
  else { ncols = 4 * s1; ktap = s0; }
  const int cin_tensor = (kind == 2 || kind == 5) ? ktap / 2 : ktap;
  const int KC = pick_kc(use_tc_ != 0, x3, ktap);
  if (ktap % KC) { seterr("channel count not a multiple of the K-block"); return IDEQ_E_INVALID; }
  std::vector<float> B = gemm_weights(kind, w, shp, KC, ncols, ntaps, ktap);
  ConvGeom g = make_geom(kind, N, Hin, Win, cin_tensor, ncols, KC, ktap, epi);
  const size_t esz = precision == IDEQ_PREC_BF16 ? 2 : 4;
  void* dW = nullptr;
  void* dWlo = nullptr;
  if (cudaMalloc(&dW, B.size() * esz) != cudaSuccess) { seterr("cudaMalloc"); return IDEQ_E_NOMEM; }
  if (precision == IDEQ_PREC_BF16) {
    std::vector<uint16_t> hb(B.size());
    for (size_t i = 0; i < B.size(); ++i) hb[i] = f2bf(B[i]);
    cudaMemcpy(dW, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice);
  } else if (x3) {
    std::vector<float> hi(B.size()), lo(B.size());
    for (size_t i = 0; i < B.size(); ++i) { hi[i] = tf32_rna(B[i]); lo[i] = tf32_rna(B[i] - hi[i]); }
    if (cudaMalloc(&dWlo, B.size() * 4) != cudaSuccess) { seterr("cudaMalloc"); cudaFree(dW); return IDEQ_E_NOMEM; }
    cudaMemcpy(dW, hi.data(), hi.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dWlo, lo.data(), lo.size() * 4, cudaMemcpyHostToDevice);
  } else {
    cudaMemcpy(dW, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  }
  int rc = IDEQ_OK;
  if (use_tc_) {
    if (!tc_supported(g, x3)) { seterr("geometry unsupported by tcgen05 path"); cudaFree(dW); cudaFree(dWlo); return IDEQ_E_UNSUPPORTED; }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    char e2[256] = {0};
    TcPlan* plan = tc_make_plan(g, x3, in, dW, dWlo, out, aux, sms, e2, sizeof(e2));
    if (!plan) { seterr(e2); cudaFree(dW); cudaFree(dWlo); return IDEQ_E_CUDA; }
    tc_launch(plan, 0);
    tc_free_plan(plan);
  } else if (precision == IDEQ_PREC_BF16) {
    launch_conv_simt<__nv_bfloat16>(g, (const __nv_bfloat16*)in, (const __nv_bfloat16*)dW, (__nv_bfloat16*)out,
                                    (const __nv_bfloat16*)aux, 0);
  } else {
    launch_conv_simt<float>(g, (const float*)in, (const float*)dW, (float*)out, (const float*)aux, 0);
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) { seterr(cudaGetErrorString(e)); rc = IDEQ_E_CUDA; }
  cudaFree(dW);
  if (dWlo) cudaFree(dWlo);
  return rc;
}

int ideq_debug_rb(int vjp, const float* wA, const float* wB, int N, int H, int W, const void* x, void* out, void* act,
                  char* err, int errlen) {
  auto seterr = [&](const char* m) { if (err && errlen > 0) { snprintf(err, errlen, "%s", m); } };
  if (!wA || !wB || !x || !out || !act || N < 1 || H < 1) { seterr("bad arguments"); return IDEQ_E_INVALID; }
  if (!rbf_supported(W, 32)) { seterr("fused residual block: W must be 128 or 256"); return IDEQ_E_UNSUPPORTED; }
  init_kernel_attributes();
  const int kind = vjp ? 1 : 0;
  const float* w1 = vjp ? wB : wA;
  const float* w2 = vjp ? wA : wB;
  void* dW[2] = {nullptr, nullptr};
  int rc = IDEQ_OK;
  for (int i = 0; i < 2 && rc == IDEQ_OK; ++i) {
    int ncols = 0, ntaps = 0, ktap = 0;
    std::vector<float> B = gemm_weights(kind, i == 0 ? w1 : w2, {32, 32, 3, 3}, 32, ncols, ntaps, ktap);
    std::vector<uint16_t> hb(B.size());
    for (size_t k = 0; k < B.size(); ++k) hb[k] = f2bf(B[k]);
    if (cudaMalloc(&dW[i], hb.size() * 2) != cudaSuccess) { seterr("cudaMalloc"); rc = IDEQ_E_NOMEM; break; }
    cudaMemcpy(dW[i], hb.data(), hb.size() * 2, cudaMemcpyHostToDevice);
  }
  if (rc == IDEQ_OK) {
    ConvGeom g = make_geom(kind, N, H, W, 32, 32, 32, 32, EPI_STORE);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    char e2[256] = {0};
    RbfPlan* plan = rbf_make_plan(vjp != 0, N, H, W, g.dh, g.dw, g.dh, g.dw, (const __nv_bfloat16*)dW[0],
                                  (const __nv_bfloat16*)dW[1], x, out, act, sms, e2, sizeof(e2));
    if (!plan) { seterr(e2); rc = IDEQ_E_CUDA; }
    else {
      rbf_launch(plan, 0);
      cudaError_t e = cudaDeviceSynchronize();
      if (e == cudaSuccess) e = cudaGetLastError();
      if (e != cudaSuccess) { seterr(cudaGetErrorString(e)); rc = IDEQ_E_CUDA; }
      rbf_free_plan(plan);
    }
  }
  for (int i = 0; i < 2; ++i) if (dW[i]) cudaFree(dW[i]);
  return rc;
}

int ideq_debug_set_fusion(ideq_ctx* ctx, int on) {
  if (!ctx) return IDEQ_E_INVALID;
  ctx->fuse_rb = on != 0;
  for (auto& kv : ctx->progs)
    for (auto& L : kv.second.layers) { if (L.plan) tc_free_plan(L.plan); if (L.i2f) img2feat_free_plan(L.i2f); if (L.rbf) rbf_free_plan(L.rbf); }
  ctx->progs.clear();
  ctx->graph_key.clear();
  return IDEQ_OK;
}

void ideq_destroy(ideq_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->gexec_plain) cudaGraphExecDestroy(ctx->gexec_plain);
  if (ctx->gexec_check) cudaGraphExecDestroy(ctx->gexec_check);
  for (auto& kv : ctx->progs)
    for (auto& L : kv.second.layers) { if (L.plan) tc_free_plan(L.plan); if (L.i2f) img2feat_free_plan(L.i2f); if (L.rbf) rbf_free_plan(L.rbf); }
  for (auto& a : ctx->allocs) cudaFree(a.p);
  for (auto& kv : ctx->jfb_plans) tc_free_plan(kv.second);
  for (auto& b : ctx->jfb_pool) cudaFree(b.first);
  if (ctx->jfb_ws) cudaFree(ctx->jfb_ws);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
  if (ctx->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(ctx->comm);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

}  // extern "C"
