// CUDA-core (FFMA) convolutions:
//   * conv_simt_kernel: the implicit GEMM of every wide layer (3x3, 2x2-patch and
//     1x1-scatter geometries of ConvGeom) -- the fp32 parity-mode path;
//   * img2feat / feat2img: the narrow head/tail 3x3 convs between the C = 1/3
//     channel image (NCHW fp32) and the w0-channel features (NHWC), used by both
//     precisions (AI ~ 20 F/B: memory-bound, no tensor-core benefit).
#include "common.cuh"
#include "kernels.h"

namespace ideq {

// ------------------------------------------------------------------ implicit GEMM (FFMA)
// Tile: BM output pixels (128: the R x Wt pixel tile the tcgen05 path uses; 32 for small grids
// such as the one-image C1 config, so the launch spreads over 4x more SMs) x BN GEMM columns
// (64, or 128 for layers with >= 128 columns: 8 x 8 register blocks, a third fewer shared loads
// per FMA); 256 threads, BM/16 pixels x BN/16 columns each; K staged 16 channels at a time.
constexpr int SM_BN = 64, SM_BK = 16;

// 16-byte vector of consecutive channels -> floats
template <typename T> struct Vec16;
template <> struct Vec16<float> {
  static constexpr int N = 4;
  static __device__ __forceinline__ void ld(const float* p, float* v) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  }
};
template <> struct Vec16<__nv_bfloat16> {
  static constexpr int N = 8;
  static __device__ __forceinline__ void ld(const __nv_bfloat16* p, float* v) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) { const float2 f = __bfloat1622float2(h[e]); v[2 * e] = f.x; v[2 * e + 1] = f.y; }
  }
};

template <typename T, int BM, int BN = SM_BN>
__global__ void __launch_bounds__(256) conv_simt_kernel(ConvGeom g, const T* __restrict__ in,
                                                        const T* __restrict__ wB, T* __restrict__ out,
                                                        const T* __restrict__ aux) {
  pdl_enter();
  constexpr int PX = BM / 16;          // pixels per thread (compute) = channels per thread (A load)
  __shared__ __align__(16) float As[SM_BK][BM + 4];
  constexpr int CPT = BN / 16;         // columns per thread (compute) = k-values per thread (B load)
  __shared__ __align__(16) float Bs[SM_BK][BN + 4];
  const int tid = threadIdx.x;
  const int mt = blockIdx.x;
  const int n0 = blockIdx.y * BN;
  const int per_img = g.tiles_h * g.tiles_w;
  const int img = mt / per_img;
  const int th = (mt % per_img) / g.tiles_w, tw = mt % g.tiles_w;
  const int oh0 = th * g.R, ow0 = tw * g.Wt;
  const int tile_px = g.R * g.Wt;

  // A-load role: 16-byte vectors of VEC consecutive channels; vector v = tid + q * 256 holds
  // channels (v % CPV) * VEC .. of tile pixel v / CPV, so a warp reads whole 32-byte sectors of
  // neighbouring pixels (one scalar load per channel at a pixel stride left 1 of 8 bytes used)
  constexpr int VEC = Vec16<T>::N, CPV = SM_BK / VEC, NVEC = BM * CPV, VPT = (NVEC + 255) / 256;
  int vpx[VPT], vcg[VPT], voh[VPT], vow[VPT];
  bool vok[VPT];
#pragma unroll
  for (int q = 0; q < VPT; ++q) {
    const int v = tid + q * 256;
    vpx[q] = v / CPV;
    vcg[q] = (v % CPV) * VEC;
    voh[q] = oh0 + vpx[q] / g.Wt;
    vow[q] = ow0 + vpx[q] % g.Wt;
    vok[q] = v < NVEC && vpx[q] < tile_px && voh[q] < g.OH && vow[q] < g.OW;
  }
  // B-load role: column bcol, CPT k-values starting at bk
  const int bcol = tid / (16 / CPT), bk = (tid % (16 / CPT)) * CPT;
  const bool bvalid = (n0 + bcol) < g.ncols;

  // compute role
  const int ty = tid >> 4, tx = tid & 15;
  float acc[PX][CPT];
#pragma unroll
  for (int i = 0; i < PX; ++i)
#pragma unroll
    for (int j = 0; j < CPT; ++j) acc[i][j] = 0.f;

  // K loop over (tap, chunk, 16-channel slice) steps, software-pipelined: the next step's
  // operands are loaded into registers while this step's products run from shared memory, so
  // the global-load latency is paid once instead of per step (the small-grid / latency-bound
  // cases: C1, the JFB tape passes)
  const int nkb = g.ntaps * g.nchunk, nkk = g.KC / SM_BK, nsteps = nkb * nkk;
  float ra[VPT][VEC], rb[CPT];
  auto load_step = [&](int st) {
    const int kb = st / nkk, kk = (st - kb * nkk) * SM_BK;
    const int tap = kb / g.nchunk, chunk = kb - tap * g.nchunk;
#pragma unroll
    for (int q = 0; q < VPT; ++q) {
      const int ih = voh[q] + g.dh[tap], iw = vow[q] + g.dw[tap];
      if (vok[q] && ih >= 0 && ih < g.inH && iw >= 0 && iw < g.inW) {
        const T* src = in + ((((long long)img * g.inH + ih) * g.inP + g.dp[tap]) * g.inW + iw) * g.inC + chunk * g.KC;
        Vec16<T>::ld(src + kk + vcg[q], ra[q]);
      } else {
#pragma unroll
        for (int e = 0; e < VEC; ++e) ra[q][e] = 0.f;
      }
    }
    const T* wsrc = wB + ((long long)kb * g.ncols + n0 + bcol) * g.KC;
    if constexpr (sizeof(T) == 4 && CPT % 4 == 0) {  // fp32 weights: 16-byte loads
#pragma unroll
      for (int j = 0; j < CPT; j += 4) {
        if (bvalid) Vec16<T>::ld(wsrc + kk + bk + j, rb + j);
        else rb[j] = rb[j + 1] = rb[j + 2] = rb[j + 3] = 0.f;
      }
    } else {
#pragma unroll
      for (int j = 0; j < CPT; ++j) rb[j] = bvalid ? ElemOps<T>::ld(wsrc + kk + bk + j) : 0.f;
    }
  };
  if (nsteps > 0) load_step(0);
  for (int st = 0; st < nsteps; ++st) {
#pragma unroll
    for (int q = 0; q < VPT; ++q)
      if (tid + q * 256 < NVEC) {
#pragma unroll
        for (int e = 0; e < VEC; ++e) As[vcg[q] + e][vpx[q]] = ra[q][e];
      }
#pragma unroll
    for (int j = 0; j < CPT; ++j) Bs[bk + j][bcol] = rb[j];
    __syncthreads();
    if (st + 1 < nsteps) load_step(st + 1);
#pragma unroll
    for (int k = 0; k < SM_BK; ++k) {
      float av[PX];
      if constexpr (PX % 4 == 0) {
#pragma unroll
        for (int i = 0; i < PX; i += 4) {
          const float4 a4 = *reinterpret_cast<const float4*>(&As[k][ty * PX + i]);
          av[i] = a4.x; av[i + 1] = a4.y; av[i + 2] = a4.z; av[i + 3] = a4.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < PX; i += 2) {
          const float2 a2 = *reinterpret_cast<const float2*>(&As[k][ty * PX + i]);
          av[i] = a2.x;
          av[i + 1] = a2.y;
        }
      }
      float bv[CPT];
      if constexpr (CPT % 4 == 0) {
#pragma unroll
        for (int j = 0; j < CPT; j += 4) {
          const float4 b = *reinterpret_cast<const float4*>(&Bs[k][tx * CPT + j]);
          bv[j] = b.x; bv[j + 1] = b.y; bv[j + 2] = b.z; bv[j + 3] = b.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < CPT; j += 2) {
          const float2 b = *reinterpret_cast<const float2*>(&Bs[k][tx * CPT + j]);
          bv[j] = b.x; bv[j + 1] = b.y;
        }
      }
#pragma unroll
      for (int i = 0; i < PX; ++i)
#pragma unroll
        for (int j = 0; j < CPT; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  // epilogue
#pragma unroll
  for (int i = 0; i < PX; ++i) {
    const int px = ty * PX + i;
    const int oh = oh0 + px / g.Wt, ow = ow0 + px % g.Wt;
    if (px >= tile_px || oh >= g.OH || ow >= g.OW) continue;
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      const int col = n0 + tx * CPT + j;
      if (col >= g.ncols) continue;
      const long long o = out_offset(g, img, oh, ow, col);
      const float av = (g.epi == EPI_RESADD || g.epi == EPI_SIGMUL) ? ElemOps<T>::ld(aux + o) : 0.f;
      ElemOps<T>::st(out + o, apply_epi(g.epi, acc[i][j], av));
    }
  }
}

template <typename T>
void launch_conv_simt(const ConvGeom& g, const T* in, const T* wB, T* out, const T* aux, cudaStream_t s) {
  const int nct = (g.ncols + SM_BN - 1) / SM_BN;
  if ((long long)g.N * g.tiles_h * g.tiles_w * nct < 2 * 148) {  // small grid: 32-pixel tiles
    ConvGeom g2 = g;
    g2.Wt = g.OW < 32 ? g.OW : 32;
    g2.R = 32 / g2.Wt;
    if (g2.R > g.OH) g2.R = g.OH;
    if (g2.R < 1) g2.R = 1;
    g2.tiles_h = (g.OH + g2.R - 1) / g2.R;
    g2.tiles_w = (g.OW + g2.Wt - 1) / g2.Wt;
    launch_k(conv_simt_kernel<T, 32>, dim3(g2.N * g2.tiles_h * g2.tiles_w, nct), 256, 0, s, g2, in, wB, out, aux);
    return;
  }
  if (g.ncols == 32) {  // 32-column layers: 256-pixel tiles (16 x 2 per thread), no idle columns
    ConvGeom g2 = g;
    g2.Wt = g.OW < 256 ? g.OW : 256;
    g2.R = 256 / g2.Wt;
    if (g2.R > g.OH) g2.R = g.OH;
    if (g2.R < 1) g2.R = 1;
    g2.tiles_h = (g.OH + g2.R - 1) / g2.R;
    g2.tiles_w = (g.OW + g2.Wt - 1) / g2.Wt;
    launch_k(conv_simt_kernel<T, 256, 32>, dim3(g2.N * g2.tiles_h * g2.tiles_w, 1), 256, 0, s, g2, in, wB, out, aux);
    return;
  }
  if (g.ncols >= 128 && g.ncols % 128 == 0) {  // wide layers: 128-column tiles, 8 x 8 per thread
    launch_k(conv_simt_kernel<T, 128, 128>, dim3(g.N * g.tiles_h * g.tiles_w, g.ncols / 128), 256, 0, s, g, in, wB,
             out, aux);
    return;
  }
  launch_k(conv_simt_kernel<T, 128>, dim3(g.N * g.tiles_h * g.tiles_w, nct), 256, 0, s, g, in, wB, out, aux);
}

// ------------------------------------------------------------------ vector helpers
// 8 consecutive channels <-> 8 floats (16 B of bf16 or 32 B of fp32)
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&v)[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int e = 0; e < 4; ++e) { const float2 f = __bfloat1622float2(h[e]); v[2 * e] = f.x; v[2 * e + 1] = f.y; }
}
__device__ __forceinline__ void load8(const float* p, float (&v)[8]) {
  const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float (&v)[8]) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}
__device__ __forceinline__ void store8(float* p, const float (&v)[8]) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}

// ------------------------------------------------------------------ head-side: image -> features
// out[n,h,w,co] = epi( sum_{ci,a,b} w_t[co][ci][a][b] in[n,ci,h+a-1,w+b-1] ), zero padding.
// A block covers 16 x 32 output pixels; the (C x 34 x 18) input halo tile is staged in shared
// memory; each thread owns two pixels (rows ty, ty+16) so every broadcast weight load feeds
// 8 FMAs (the kernel is otherwise limited by shared-memory issue, not FMA).
constexpr int HT_ROWS = 32;
template <typename T, int WO, int C>
__global__ void __launch_bounds__(256) img2feat_kernel(const float* __restrict__ in, const float* __restrict__ w_t,
                                                       T* __restrict__ out, const T* __restrict__ aux, int epi,
                                                       int N, int H, int W) {
  __shared__ __align__(16) float wsm[3 * 9][WO];
  __shared__ float tile[3][HT_ROWS + 2][18 + 1];
  // the weights (constant since create) are staged before waiting for the predecessor grid
  for (int t = threadIdx.x; t < WO * C * 9; t += blockDim.x) {
    const int co = t / (C * 9), r = t % (C * 9);
    wsm[r][co] = w_t[t];  // [ci*9 + a*3 + b][co]
  }
  pdl_enter();
  const int n = blockIdx.z, h0 = blockIdx.y * HT_ROWS, w0 = blockIdx.x * 16;
  const long long HW = (long long)H * W;
  for (int t = threadIdx.x; t < C * (HT_ROWS + 2) * 18; t += blockDim.x) {
    const int ci = t / ((HT_ROWS + 2) * 18), q = t % ((HT_ROWS + 2) * 18), u = q / 18, v = q % 18;
    const int hh = h0 + u - 1, ww = w0 + v - 1;
    tile[ci][u][v] = (hh >= 0 && hh < H && ww >= 0 && ww < W) ? in[((long long)n * C + ci) * HW + (long long)hh * W + ww] : 0.f;
  }
  __syncthreads();
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  const int w = w0 + tx;
  constexpr int G = WO < 32 ? WO : 32;  // outputs per register group (keeps acc in registers)
#pragma unroll 1
  for (int g0 = 0; g0 < WO; g0 += G) {
    float acc[2][G];
#pragma unroll
    for (int co = 0; co < G; ++co) { acc[0][co] = 0.f; acc[1][co] = 0.f; }
#pragma unroll
    for (int ci = 0; ci < C; ++ci) {  // C is a template constant: the 9*C taps unroll fully
#pragma unroll
      for (int a = 0; a < 3; ++a) {
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          const float v0 = tile[ci][ty + a][tx + b];
          const float v1 = tile[ci][ty + 16 + a][tx + b];
          const float4* wr = reinterpret_cast<const float4*>(wsm[ci * 9 + a * 3 + b] + g0);
#pragma unroll
          for (int c4 = 0; c4 < G / 4; ++c4) {
            const float4 w4 = wr[c4];
            acc[0][4 * c4] = fmaf(w4.x, v0, acc[0][4 * c4]);
            acc[0][4 * c4 + 1] = fmaf(w4.y, v0, acc[0][4 * c4 + 1]);
            acc[0][4 * c4 + 2] = fmaf(w4.z, v0, acc[0][4 * c4 + 2]);
            acc[0][4 * c4 + 3] = fmaf(w4.w, v0, acc[0][4 * c4 + 3]);
            acc[1][4 * c4] = fmaf(w4.x, v1, acc[1][4 * c4]);
            acc[1][4 * c4 + 1] = fmaf(w4.y, v1, acc[1][4 * c4 + 1]);
            acc[1][4 * c4 + 2] = fmaf(w4.z, v1, acc[1][4 * c4 + 2]);
            acc[1][4 * c4 + 3] = fmaf(w4.w, v1, acc[1][4 * c4 + 3]);
          }
        }
      }
    }
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const int h = h0 + ty + 16 * p;
      if (h >= H || w >= W) continue;
      const long long pix = (long long)n * HW + (long long)h * W + w;
      T* o = out + pix * WO + g0;
      const T* x = aux ? aux + pix * WO + g0 : nullptr;
#pragma unroll
      for (int c8 = 0; c8 < G; c8 += 8) {
        float v[8], av[8];
        if (x) load8(x + c8, av);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = apply_epi(epi, acc[p][c8 + e], x ? av[e] : 0.f);
        store8(o + c8, v);
      }
    }
  }
}

template <typename T>
void launch_img2feat(const float* in, const float* w_t, T* out, const T* aux, int epi, int N, int C, int H, int W,
                     int wout, cudaStream_t s) {
  dim3 grid((W + 15) / 16, (H + HT_ROWS - 1) / HT_ROWS, N);
#define I2F(WO)                                                                                          \
  case WO:                                                                                               \
    if (C == 1) launch_k(img2feat_kernel<T, WO, 1>, grid, 256, 0, s, in, w_t, out, aux, epi, N, H, W);         \
    else launch_k(img2feat_kernel<T, WO, 3>, grid, 256, 0, s, in, w_t, out, aux, epi, N, H, W);                \
    break;
  switch (wout) {
    I2F(16) I2F(32) I2F(64)
    default: break;  // rejected by the runtime at create
  }
#undef I2F
}

// ------------------------------------------------------------------ tail-side: features -> image
// out[n,c,h,w] = sum_{ci,a,b} w_t[c][ci][a][b] in[n,h+a-1,w+b-1,ci] + alpha * aux[n,c,h,w]
// A block covers 16 x 32 output pixels (two per thread, rows ty and ty+16); the 34x18xWI input
// tile is loaded with 16-byte vectors and kept as fp32 with a padded pixel stride (WI+4 floats)
// so float4 reads are conflict-free; weights are float4 (c0, c1, c2, 0) broadcasts.
template <typename T, int WI>
__global__ void __launch_bounds__(256) feat2img_kernel(const T* __restrict__ in, const float* __restrict__ w_t,
                                                       float* __restrict__ out, const float* __restrict__ aux,
                                                       float alpha, int N, int C, int H, int W) {
  extern __shared__ __align__(16) float smf[];
  constexpr int PS = WI + 4;
  float4* wsm = reinterpret_cast<float4*>(smf);  // [9][WI] : (a*3+b, ci) -> (c0, c1, c2, 0)
  float* tile = smf + 9 * WI * 4;                 // [(HT_ROWS+2)*18][PS]
  const int n = blockIdx.z;
  const int h0 = blockIdx.y * HT_ROWS, w0 = blockIdx.x * 16;
  for (int t = threadIdx.x; t < 9 * WI; t += blockDim.x) {
    const int ab = t / WI, ci = t % WI;
    float4 w4;
    w4.x = w_t[(0 * WI + ci) * 9 + ab];
    w4.y = C > 1 ? w_t[(1 * WI + ci) * 9 + ab] : 0.f;
    w4.z = C > 1 ? w_t[(2 * WI + ci) * 9 + ab] : 0.f;
    w4.w = 0.f;
    wsm[t] = w4;
  }
  pdl_enter();  // weights staged; now wait for the producer of `in`
  constexpr int V = WI / 8;  // 8-channel vectors per pixel
  for (int t = threadIdx.x; t < (HT_ROWS + 2) * 18 * V; t += blockDim.x) {
    const int q = t / V, c8 = (t % V) * 8;
    const int u = q / 18, v = q % 18;
    const int hh = h0 + u - 1, ww = w0 + v - 1;
    float f[8];
    if (hh >= 0 && hh < H && ww >= 0 && ww < W) {
      load8(in + (((long long)n * H + hh) * W + ww) * WI + c8, f);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) f[e] = 0.f;
    }
    float* dst = tile + q * PS + c8;
    *reinterpret_cast<float4*>(dst) = make_float4(f[0], f[1], f[2], f[3]);
    *reinterpret_cast<float4*>(dst + 4) = make_float4(f[4], f[5], f[6], f[7]);
  }
  __syncthreads();
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  const int w = w0 + tx;
  float acc[2][3] = {{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const float* tp0 = tile + ((ty + a) * 18 + (tx + b)) * PS;
      const float* tp1 = tp0 + 16 * 18 * PS;
      const float4* wp = wsm + (a * 3 + b) * WI;
#pragma unroll
      for (int ci = 0; ci < WI; ci += 4) {  // fully unrolled: loads hoist ahead of their FMAs
        const float4 v0 = *reinterpret_cast<const float4*>(tp0 + ci);
        const float4 v1 = *reinterpret_cast<const float4*>(tp1 + ci);
        const float a0[4] = {v0.x, v0.y, v0.z, v0.w};
        const float a1[4] = {v1.x, v1.y, v1.z, v1.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float4 ww = wp[ci + e];
          acc[0][0] = fmaf(ww.x, a0[e], acc[0][0]);
          acc[0][1] = fmaf(ww.y, a0[e], acc[0][1]);
          acc[0][2] = fmaf(ww.z, a0[e], acc[0][2]);
          acc[1][0] = fmaf(ww.x, a1[e], acc[1][0]);
          acc[1][1] = fmaf(ww.y, a1[e], acc[1][1]);
          acc[1][2] = fmaf(ww.z, a1[e], acc[1][2]);
        }
      }
    }
  }
  const long long HW = (long long)H * W;
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const int h = h0 + ty + 16 * p;
    if (h >= H || w >= W) continue;
    const long long o0 = (long long)n * C * HW + (long long)h * W + w;
    out[o0] = acc[p][0] + (aux ? alpha * aux[o0] : 0.f);
    if (C > 1) {
      out[o0 + HW] = acc[p][1] + (aux ? alpha * aux[o0 + HW] : 0.f);
      out[o0 + 2 * HW] = acc[p][2] + (aux ? alpha * aux[o0 + 2 * HW] : 0.f);
    }
  }
}

template <typename T>
void launch_feat2img(const T* in, const float* w_t, float* out, const float* aux, float alpha, int N, int C, int H,
                     int W, int win, cudaStream_t s) {
  dim3 grid((W + 15) / 16, (H + HT_ROWS - 1) / HT_ROWS, N);
  const size_t sm = sizeof(float) * (9 * 4 * win + (HT_ROWS + 2) * 18 * (win + 4));
  switch (win) {
    case 16: launch_k(feat2img_kernel<T, 16>, grid, 256, sm, s, in, w_t, out, aux, alpha, N, C, H, W); break;
    case 32: launch_k(feat2img_kernel<T, 32>, grid, 256, sm, s, in, w_t, out, aux, alpha, N, C, H, W); break;
    case 64: launch_k(feat2img_kernel<T, 64>, grid, 256, sm, s, in, w_t, out, aux, alpha, N, C, H, W); break;
    default: break;
  }
}

void init_attrs_simt() {
  set_max_dyn_smem(feat2img_kernel<float, 16>);
  set_max_dyn_smem(feat2img_kernel<float, 32>);
  set_max_dyn_smem(feat2img_kernel<float, 64>);
  set_max_dyn_smem(feat2img_kernel<__nv_bfloat16, 16>);
  set_max_dyn_smem(feat2img_kernel<__nv_bfloat16, 32>);
  set_max_dyn_smem(feat2img_kernel<__nv_bfloat16, 64>);
}

template void launch_conv_simt<float>(const ConvGeom&, const float*, const float*, float*, const float*, cudaStream_t);
template void launch_conv_simt<__nv_bfloat16>(const ConvGeom&, const __nv_bfloat16*, const __nv_bfloat16*,
                                              __nv_bfloat16*, const __nv_bfloat16*, cudaStream_t);
template void launch_img2feat<float>(const float*, const float*, float*, const float*, int, int, int, int, int, int,
                                     cudaStream_t);
template void launch_img2feat<__nv_bfloat16>(const float*, const float*, __nv_bfloat16*, const __nv_bfloat16*, int,
                                             int, int, int, int, int, cudaStream_t);
template void launch_feat2img<float>(const float*, const float*, float*, const float*, float, int, int, int, int, int,
                                     cudaStream_t);
template void launch_feat2img<__nv_bfloat16>(const __nv_bfloat16*, const float*, float*, const float*, float, int,
                                             int, int, int, int, cudaStream_t);

}  // namespace ideq
