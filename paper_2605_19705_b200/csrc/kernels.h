// Internal kernel launch interface (not part of the public C ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>
#include "common.cuh"

namespace ideq {

enum StepMode : int { STEP_PROX_INPAINT = 0, STEP_GRAD_BUF = 1, STEP_GRAD_INPAINT = 2, STEP_X1_BUF = 3, STEP_GRAD_RICIAN = 4, STEP_GRAD_MRI = 5 };

struct StepArgs {
  int N, C, H, W;
  long long d;            // C*H*W
  int parts;              // partial-sum slots per image
  const float* z;         // z^k (read)
  float* zout;            // z^{k+1} (written; may alias z)
  const float* gg;        // grad g(z^k)
  const float* y;         // observation
  float* X0;              // iterate ping-pong buffers: x^k = X[k&1], x^{k+1} = X[(k+1)&1]
  float* X1;
  const uint8_t* mask;    // inpainting mask [N][H][W]
  float* fbuf;            // fidelity scratch (A z - y, grad f or x^{k+1})
  float* fbuf2;           // second scratch (A^T y)
  const float* kern;      // blur kernel(s)
  int ksize, kernel_per_image;
  float lam, tau, beta;
  float inv_s2;           // Rician: 1 / sigma^2
  const int* active;      // [N]
  const int* kdev;        // iteration counter k
  float* partials;        // [N][parts][3]
};

struct FinalizeArgs {
  int N, parts, check_every, stop_rule;
  float tol;
  const float* partials;
  int* active;
  int* status;
  int* iters;
  float* res;
  float* r_now;
  float* trace;   // [trace_cap] or null: max_i r_i of iteration k < trace_cap
  int trace_cap;
  float* rmax;    // 1 float (NCCL all-reduce target)
  int* n_active;
  int* act_list;  // [N] compacted indices of the active images (first *n_active), for the conv tile loops
  int* kdev;
  // NEXT-1: restart (Eq. 5) and averaging (Alg. 1/2 steps 12-13)
  int restart;        // 0 off, 1 Alg. 1 semantics, 2 Alg. 2 semantics
  double B2;          // restart_B^2
  int averaging, K;   // K = max_iter
  int* rk;            // [N] iterations since the last (Alg. 1) restart
  double* rsum;       // [N] sum of ||x^{t+1} - x^t||^2 since then
  int* flags;         // [N] bit0 stepped this iteration, bit1 restart, bit2 new averaging minimum
  int* nrest;         // [N] restart count
  float* best;        // [N] smallest increment in the averaging window so far
  int* k0;            // [N] its iteration index (-1: none)
};

struct PostArgs {
  int N;
  long long d;
  const int* flags;
  const int* kdev;
  float* X0;
  float* X1;
  float* Z;      // z^{k+1} (restart: := x^{k+1})
  float* Zsum;   // running sum of z^0..z^k (averaging) or null
  float* Xsnap;  // averaging snapshot mean(z^0..z^K0)
};

// ---- batched 2-D FFT passes (fft.cu)
struct FftArgs {
  int C, H, W, J, logH, logW;
  const float2* tw_h;   // exp(-2 pi i k / H), k < H/2
  const float2* tw_w;   // exp(-2 pi i k / W), k < W/2
  float2* spec;         // blur: [N][C][H][W/2+1]; phase: [N][J][H][W]
  const float* z;       // prox rhs / phase input
  const float* gg;
  const float* aty;
  float tau, lam;
  const float* dgl;     // [H][W/2+1] 1 / (1 + tau |K^|^2)
  const float2* khat;   // [H][W/2+1]
  const float2* pmask;  // [J][H][W]
  const float* y;       // phase observations [N][J][H][W]
  const int* active;
};
bool fft_size_ok(int H, int W);
void fft_fill_args(FftArgs& f);
int fft_parts_per_image(int C, int H, int W);
int phase_parts_per_image(int H, int W, int J);  // J = number of phase masks
void launch_blur_rows_fwd(const FftArgs& f, const float* src, int mode, int N, cudaStream_t s);
void launch_blur_cols(const FftArgs& f, int op, int N, cudaStream_t s);
struct StepArgs;
void launch_blur_rows_inv(const FftArgs& f, const StepArgs& a, float* dst, int mode, int N, cudaStream_t s);
void launch_embed_kernel(const float* k, int ks, float* plane, int H, int W, cudaStream_t s);
void launch_blur_diag(const float2* khat, float tau, float* dgl, int n, cudaStream_t s);
void launch_phase_rows_fwd(const FftArgs& f, int N, cudaStream_t s);
void launch_phase_cols(const FftArgs& f, int N, cudaStream_t s);
void launch_phase_rows_inv(const FftArgs& f, const StepArgs& a, float* dst, int mode, int N, cudaStream_t s);
void init_attrs_fft();

void launch_pointwise_step(int mode, const StepArgs& a, cudaStream_t s);
int blur_parts_per_image(int C, int H, int W, int ks);  // residual partials of the direct blur step
void launch_blur_residual(const StepArgs& a, cudaStream_t s);
void launch_blur_adjoint(int mode, const StepArgs& a, const float* src, cudaStream_t s);
void launch_finalize(const FinalizeArgs& f, cudaStream_t s);
void launch_advance_a(const FinalizeArgs& f, cudaStream_t s);
void launch_advance_b(const FinalizeArgs& f, cudaStream_t s);
void launch_init_state(const FinalizeArgs& f, cudaStream_t s);
void launch_gather(const int* iters, const float* X1, float* X0, int N, long long d, cudaStream_t s);
void launch_post_step(const PostArgs& a, cudaStream_t s);
void launch_mri_fill(const float* y, const uint8_t* kmask, float2* spec, int N, int H, int W, float scale,
                     cudaStream_t s);
void launch_mri_masks(const uint8_t* kmask, float* mhalf, float* dgl, float tau, int H, int W, cudaStream_t s);
void launch_sub(const float* a, const float* b, float* out, long long n, cudaStream_t s);
// ---- JFB training gradient (jfb.cu)
size_t wgrad_workspace(const ConvGeom& g);  // floats of split partials launch_wgrad_geom needs
void launch_wgrad_geom(const ConvGeom& g, const float* in, const float* gout, float* dB, float* ws, cudaStream_t s);
size_t headtail_wgrad_workspace(int N, int C, int H, int wf);
void launch_head_wgrad(const float* img, const float* gf, float* dW, float* ws, int N, int C, int H, int W, int wf,
                       cudaStream_t s);
void launch_tail_wgrad(const float* f, const float* gimg, float* dW, float* ws, int N, int C, int H, int W, int wf,
                       cudaStream_t s);
void launch_sp_forward(const float* p, float* a, long long n, cudaStream_t s);
void launch_sp_tangent(const float* a, const float* pd, float* ad, long long n, cudaStream_t s);
void launch_sp_reverse(const float* a, const float* pd, const float* ab, const float* adb, float* pb, float* pdb,
                       long long n, cudaStream_t s);
void launch_scale(float* x, float s, long long n, cudaStream_t st);
void launch_jfb_residual(const float* z, const float* xs, const float* gg, const float* gf, const float* y,
                         const uint8_t* mask, int prox, float lam, float tau, long long n, long long HW, long long CHW,
                         float* v, float* terms, cudaStream_t s);
void launch_sums(const float* x, long long n, int k, double* part, double* out, cudaStream_t s);
void launch_rician_grad(const float* x, const float* y, float inv_s2, float* out, long long n, cudaStream_t s);
void launch_avg_out(const int* k0, const int* status, const int* iters, int K, const float* Xsnap, float* X, int N,
                    long long d, cudaStream_t s);
void launch_inpaint_grad(const float* x, const float* y, const uint8_t* m, float* out, int N, int C, int H, int W,
                         cudaStream_t s);
void launch_inpaint_prox(const float* v, const float* y, const uint8_t* m, float tau, float* out, int N, int C, int H,
                         int W, cudaStream_t s);

// ---- convolutions
// FFMA implicit GEMM (any precision; fp32 math). wB: [ntaps*nchunk][ncols][KC].
template <typename T>
void launch_conv_simt(const ConvGeom& g, const T* in, const T* wB, T* out, const T* aux, cudaStream_t s);
// C (1 or 3, NCHW fp32) -> w (NHWC T) 3x3 conv; w_t: [w][C][3][3] fp32 (already flipped for adjoints).
template <typename T>
void launch_img2feat(const float* in, const float* w_t, T* out, const T* aux, int epi, int N, int C, int H, int W,
                     int wout, cudaStream_t s);
// w (NHWC T) -> C (NCHW fp32) 3x3 conv; w_t: [C][w][3][3]; out = acc + alpha * aux (aux NCHW fp32 or null).
template <typename T>
void launch_feat2img(const T* in, const float* w_t, float* out, const float* aux, float alpha, int N, int C, int H,
                     int W, int win, cudaStream_t s);

// tcgen05 implicit GEMM, fp32 TMEM accumulators: bf16 operands, or (x3) fp32 operands as 3xTF32
// (wBlo = the lo half of the pre-split weights). Returns false / null if the geometry is
// unsupported (the runtime then refuses the configuration).
struct TcPlan;
bool tc_supported(const ConvGeom& g, bool x3);
TcPlan* tc_make_plan(const ConvGeom& g, bool x3, const void* in, const void* wB, const void* wBlo, void* out,
                     const void* aux, int num_sms, char* err, size_t errlen);
void tc_launch(const TcPlan* p, cudaStream_t s);
void tc_free_plan(TcPlan* p);
void tc_plan_set_image(TcPlan* p, float* out, const float* aux, float alpha, int C);
void tc_plan_set_active(TcPlan* p, const int* act_list, const int* n_act);  // live-image list for tile skipping
void tc_plan_enable_skip(TcPlan* p, bool on);
int tc_plan_is_halo(const TcPlan* p);
// im2col of a C-channel fp32 NCHW image into [N][H][W][32] bf16: k = c*9 + a*3 + b (zero beyond 9C)
struct I2FPlan;  // fused head: the output tensor map (conv_tc.cu)
I2FPlan* img2feat_make_plan(__nv_bfloat16* out, int N, int H, int W, int NC, char* err, size_t errlen);
void img2feat_free_plan(I2FPlan* p);
void launch_img2feat_tc(const I2FPlan* plan, const float* in, const __nv_bfloat16* wB, const int* act_list,
                        const int* n_act, int N, int C,
                        int H, int W, int NC, int num_sms, cudaStream_t s);

// Residual-block-fused level-0 convolutions (rbf.cu): forward t' = t + B sp(A t) (+ saved a) or
// VJP g' = g + A^T((B^T g) . sp'(a)), full rows of W in {128, 256} pixels, 32 channels, bf16.
struct RbfPlan;
bool rbf_supported(int W, int C);
RbfPlan* rbf_make_plan(bool vjp, int N, int H, int W, const int dh1[9], const int dw1[9], const int dh2[9],
                       const int dw2[9], const __nv_bfloat16* w1, const __nv_bfloat16* w2, const void* x, void* out,
                       void* act, int num_sms, char* err, size_t errlen);
void rbf_set_active(RbfPlan* p, const int* act_list, const int* n_act);
void rbf_enable_skip(RbfPlan* p, bool on);
void rbf_launch(const RbfPlan* p, cudaStream_t s);
void rbf_free_plan(RbfPlan* p);
void init_attrs_rbf();

// Whole-solve persistent kernel of the tiny network (tiny_solve.cu): one 8- or 16-CTA cluster per image.
struct TinySolveArgs {
  int N, H, W, ks, kper;
  const float* kern;
  const float *w1, *w2, *w3;  // c1 [16][1][3][3], c2 [16][16][3][3], c3 [1][16][3][3] (blob order)
  const float* y;
  float* x;                   // in: x^0, out: x-hat
  float lam, tau, beta, tol;
  int max_iter, check_every;
  int* iters;
  float* res;
  int* status;
  float* trace;  // zeroed by the caller
  int trace_cap;
  int* kdone;    // zeroed by the caller
};
bool tiny_solve_supported(int H, int W, int ks);
size_t tiny_solve_smem(int H, int W, int ks);
void launch_tiny_solve(const TinySolveArgs& a, cudaStream_t s);
void init_attrs_tiny();

// Raise the dynamic shared-memory limit of every kernel once (before any graph capture).
void init_kernel_attributes();
void init_attrs_simt();
void init_attrs_tc();
void init_attrs_step();

}  // namespace ideq
