// Memory-bound kernels of the i-DEQ iteration: data-fidelity passes, the fused
// update (extrapolation + fidelity step / prox + residual partials), the
// per-image residual finalize / stop logic, and the output gather.
//
// Iterate state is fp32 NCHW [N][C][H][W] in both precisions (reading Q19).
// Every kernel is deterministic: partial sums have a fixed block -> (image, part)
// assignment and are combined in a fixed order in fp64 by ideq_finalize_kernel.
#include "common.cuh"
#include "kernels.h"

namespace ideq {

// ------------------------------------------------------------------ block reduction
struct Partial3 { float d2, n2, bad; };

__device__ __forceinline__ void block_reduce_store(Partial3 v, float* out3) {
  __shared__ float red[3][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.d2 += __shfl_xor_sync(0xffffffffu, v.d2, o);
    v.n2 += __shfl_xor_sync(0xffffffffu, v.n2, o);
    v.bad += __shfl_xor_sync(0xffffffffu, v.bad, o);
  }
  if (lane == 0) { red[0][wid] = v.d2; red[1][wid] = v.n2; red[2][wid] = v.bad; }
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    Partial3 s{lane < nw ? red[0][lane] : 0.f, lane < nw ? red[1][lane] : 0.f, lane < nw ? red[2][lane] : 0.f};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s.d2 += __shfl_xor_sync(0xffffffffu, s.d2, o);
      s.n2 += __shfl_xor_sync(0xffffffffu, s.n2, o);
      s.bad += __shfl_xor_sync(0xffffffffu, s.bad, o);
    }
    if (lane == 0) { out3[0] = s.d2; out3[1] = s.n2; out3[2] = s.bad; }
  }
}

// Common tail of every update: given x^{k+1} for one element, write it, write
// z^{k+1} = x^{k+1} + beta (x^{k+1} - x^k) (Eq. 4 of the NEXT iteration, fused
// here so x^{k-1} is never re-read) and accumulate the residual partials.
__device__ __forceinline__ void tail_elem(float x1, float xk, float beta, float* xn, float* zn, Partial3& acc) {
  *xn = x1;
  *zn = x1 + beta * (x1 - xk);
  const float d = x1 - xk;
  if (isfinite(x1)) { acc.d2 += d * d; } else { acc.bad += 1.f; }
  acc.n2 += xk * xk;
}

// ------------------------------------------------------------------ Rician fidelity (App. D.3.3)
// B(t) = I1(t) / I0(t) for t >= 0 in fp32: the defining power series below t = 20 (terms
// (t/2)^{2k} / (k!)^2 stay far from fp32 overflow there), the asymptotic expansion
// 1 - 1/(2t) - 1/(8t^2) - 1/(8t^3) - 25/(128 t^4) above (|error| < 1.5e-7 at t = 20).
__device__ __forceinline__ float bessel_ratio_f(float t) {
  if (t < 20.f) {
    const float q = 0.25f * t * t;
    float a = 1.f, i0 = 1.f, i1 = 1.f;  // i1 accumulates sum a_k / (k + 1)
    for (int k = 1; k < 64; ++k) {
      a *= q / (float)(k * k);
      i0 += a;
      i1 += a / (float)(k + 1);
      if (a < 1e-9f * i0) break;
    }
    return 0.5f * t * i1 / i0;
  }
  const float r = 1.f / t;
  return 1.f - r * (0.5f + r * (0.125f + r * (0.125f + r * (25.f / 128.f))));
}
// grad f = x / sigma^2 - (y / sigma^2) B(x y / sigma^2); B is odd
__device__ __forceinline__ float rician_grad_f(float x, float y, float inv_s2) {
  const float t = x * y * inv_s2;
  const float b = bessel_ratio_f(fabsf(t));
  return x * inv_s2 - y * inv_s2 * copysignf(b, t);
}

__global__ void __launch_bounds__(256) rician_grad_kernel(const float* __restrict__ x, const float* __restrict__ y,
                                                          float inv_s2, float* __restrict__ out, long long n) {
  pdl_enter();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = rician_grad_f(x[i], y[i], inv_s2);
}

__global__ void sub_kernel(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ out,
                           long long n) {
  pdl_enter();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = a[i] - b[i];
}
void launch_sub(const float* a, const float* b, float* out, long long n, cudaStream_t s) {
  long long g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  launch_k(sub_kernel, (unsigned)g, 256, 0, s, a, b, out, n);
}

void launch_rician_grad(const float* x, const float* y, float inv_s2, float* out, long long n, cudaStream_t s) {
  long long b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  launch_k(rician_grad_kernel, (unsigned)b, 256, 0, s, x, y, inv_s2, out, n);
}

// ------------------------------------------------------------------ pointwise step kernels
// Block -> (image n, part) with `parts` blocks per image, each covering a fixed
// contiguous chunk of the image's d = C*H*W elements.
template <int MODE>
__global__ void __launch_bounds__(256) pointwise_step_kernel(StepArgs a) {
  pdl_enter();
  const int n = blockIdx.y, part = blockIdx.x;
  if (!a.active[n]) return;
  const int k = *a.kdev;
  const float* xk_base = (k & 1) ? a.X1 : a.X0;
  float* xn_base = (k & 1) ? a.X0 : a.X1;
  const long long d = a.d;
  const long long chunk = (d + a.parts - 1) / a.parts;
  const long long beg = part * chunk;
  const long long end = min(d, beg + chunk);
  const long long off = (long long)n * d;
  const long long HW = (long long)a.H * a.W;
  const uint8_t* mrow = a.mask ? a.mask + (long long)n * HW : nullptr;
  // pixel index within the channel plane, advanced incrementally (no 64-bit modulo per element)
  uint32_t pix = (uint32_t)((beg + threadIdx.x) % HW);
  Partial3 acc{0.f, 0.f, 0.f};
  for (long long e = beg + threadIdx.x; e < end; e += blockDim.x) {
    const long long i = off + e;
    const float z = a.z[i], gg = a.gg[i], xk = xk_base[i];
    float x1;
    if (MODE == STEP_PROX_INPAINT) {
      // v = z - tau lam grad g ; prox = (tau M y + v) / (tau M + 1)
      const float m = (float)mrow[pix];
      const float v = z - a.tau * a.lam * gg;
      x1 = (a.tau * m * a.y[i] + v) / (a.tau * m + 1.f);
    } else if (MODE == STEP_GRAD_BUF) {
      // x = z - tau (grad f + lam grad g), grad f precomputed in a.fbuf
      x1 = z - a.tau * (a.fbuf[i] + a.lam * gg);
    } else if (MODE == STEP_GRAD_MRI) {
      // grad f = Re F^-1 M (M F z - y) = fbuf - fbuf2 with fbuf = F^-1 M F z, fbuf2 = Re F^-1 M y
      x1 = z - a.tau * (a.fbuf[i] - a.fbuf2[i] + a.lam * gg);                   // Alg. 1 l.8
    } else if (MODE == STEP_GRAD_RICIAN) {
      x1 = z - a.tau * (rician_grad_f(z, a.y[i], a.inv_s2) + a.lam * gg);   // Alg. 1 l.8
    } else if (MODE == STEP_GRAD_INPAINT) {
      const float m = (float)mrow[pix];
      x1 = z - a.tau * (m * (m * z - a.y[i]) + a.lam * gg);
    } else {  // STEP_X1_BUF: x^{k+1} already computed (FFT prox output)
      x1 = a.fbuf[i];
    }
    tail_elem(x1, xk, a.beta, xn_base + i, a.zout + i, acc);
    pix += blockDim.x;
    while (pix >= (uint32_t)HW) pix -= (uint32_t)HW;
  }
  block_reduce_store(acc, a.partials + ((long long)n * a.parts + part) * 3);
}

// Vectorised form (every config: d and H*W multiples of 4): each thread moves float4 of z, grad g,
// x^k, y (and a uchar4 of the mask: 4 consecutive pixels of one channel plane) and writes float4
// of x^{k+1}, z^{k+1}; 32-bit indices inside the image (d < 2^31), the image offset applied once
// to the base pointers. Per element it reads 16 B (+ 1/C B of mask) and writes 8 B.
template <int MODE>
__device__ __forceinline__ float step_x1(const StepArgs& a, float z, float gg, float y, float m, float fb, float fb2) {
  if (MODE == STEP_PROX_INPAINT) {
    const float v = z - a.tau * a.lam * gg;
    return (a.tau * m * y + v) / (a.tau * m + 1.f);
  } else if (MODE == STEP_GRAD_BUF) {
    return z - a.tau * (fb + a.lam * gg);
  } else if (MODE == STEP_GRAD_MRI) {
    return z - a.tau * (fb - fb2 + a.lam * gg);              // Alg. 1 l.8, grad f = fbuf - fbuf2
  } else if (MODE == STEP_GRAD_RICIAN) {
    return z - a.tau * (rician_grad_f(z, y, a.inv_s2) + a.lam * gg);
  } else if (MODE == STEP_GRAD_INPAINT) {
    return z - a.tau * (m * (m * z - y) + a.lam * gg);
  }
  return fb;  // STEP_X1_BUF
}

template <int MODE>
__global__ void __launch_bounds__(256) pointwise_step_v4_kernel(StepArgs a) {
  pdl_enter();
  const int n = blockIdx.y, part = blockIdx.x;
  if (!a.active[n]) return;
  const int k = *a.kdev;
  constexpr bool USE_Y = MODE == STEP_PROX_INPAINT || MODE == STEP_GRAD_RICIAN || MODE == STEP_GRAD_INPAINT;
  constexpr bool USE_M = MODE == STEP_PROX_INPAINT || MODE == STEP_GRAD_INPAINT;
  constexpr bool USE_FB = MODE == STEP_GRAD_BUF || MODE == STEP_GRAD_MRI || MODE == STEP_X1_BUF;
  const long long off = (long long)n * a.d;
  const float4* z4 = reinterpret_cast<const float4*>(a.z + off);
  const float4* g4 = reinterpret_cast<const float4*>(a.gg + off);
  const float4* xk4 = reinterpret_cast<const float4*>(((k & 1) ? a.X1 : a.X0) + off);
  float4* xn4 = reinterpret_cast<float4*>(((k & 1) ? a.X0 : a.X1) + off);
  float4* zn4 = reinterpret_cast<float4*>(a.zout + off);
  const float4* y4 = USE_Y ? reinterpret_cast<const float4*>(a.y + off) : nullptr;
  const float4* f4 = USE_FB ? reinterpret_cast<const float4*>(a.fbuf + off) : nullptr;
  const float4* f24 = MODE == STEP_GRAD_MRI ? reinterpret_cast<const float4*>(a.fbuf2 + off) : nullptr;
  const uint32_t HW4 = (uint32_t)(a.H * a.W) >> 2;
  const uchar4* m4 = USE_M ? reinterpret_cast<const uchar4*>(a.mask + (long long)n * a.H * a.W) : nullptr;
  const uint32_t d4 = (uint32_t)(a.d >> 2);
  const uint32_t chunk = (d4 + a.parts - 1) / a.parts;
  const uint32_t beg = part * chunk;
  const uint32_t end = min(d4, beg + chunk);
  uint32_t pix = (beg + threadIdx.x) % HW4;  // float4 index inside the channel plane
  Partial3 acc{0.f, 0.f, 0.f};
  for (uint32_t e = beg + threadIdx.x; e < end; e += blockDim.x) {
    const float4 z = z4[e], gg = __ldg(g4 + e), xk = xk4[e];  // z^{k+1} overwrites z in place
    const float4 y = USE_Y ? __ldg(y4 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 fb = USE_FB ? f4[e] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 fb2 = MODE == STEP_GRAD_MRI ? __ldg(f24 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 m = make_float4(0.f, 0.f, 0.f, 0.f);
    if (USE_M) {
      const uchar4 mu = __ldg(m4 + pix);
      m = make_float4((float)mu.x, (float)mu.y, (float)mu.z, (float)mu.w);
    }
    float4 x1, zn;
    x1.x = step_x1<MODE>(a, z.x, gg.x, y.x, m.x, fb.x, fb2.x);
    x1.y = step_x1<MODE>(a, z.y, gg.y, y.y, m.y, fb.y, fb2.y);
    x1.z = step_x1<MODE>(a, z.z, gg.z, y.z, m.z, fb.z, fb2.z);
    x1.w = step_x1<MODE>(a, z.w, gg.w, y.w, m.w, fb.w, fb2.w);
    // z^{k+1} = x^{k+1} + beta (x^{k+1} - x^k) (Eq. 4 of the next iteration) and the residual partials
    const float dx = x1.x - xk.x, dy = x1.y - xk.y, dz = x1.z - xk.z, dw = x1.w - xk.w;
    zn = make_float4(x1.x + a.beta * dx, x1.y + a.beta * dy, x1.z + a.beta * dz, x1.w + a.beta * dw);
    xn4[e] = x1;
    zn4[e] = zn;
    if (isfinite(x1.x) && isfinite(x1.y) && isfinite(x1.z) && isfinite(x1.w)) {
      acc.d2 += dx * dx + dy * dy + dz * dz + dw * dw;
    } else {
      acc.bad += 1.f;
    }
    acc.n2 += xk.x * xk.x + xk.y * xk.y + xk.z * xk.z + xk.w * xk.w;
    pix += blockDim.x;
    while (pix >= HW4) pix -= HW4;
  }
  block_reduce_store(acc, a.partials + ((long long)n * a.parts + part) * 3);
}

// ------------------------------------------------------------------ direct periodic blur
// (A x)[m,n] = sum_{i,j} k[i,j] x[(m-i+kc) mod H, (n-j+kc) mod W]   (true convolution, Q8)
// (A^T r)[m,n] = sum_{i,j} k[i,j] r[(m+i-kc) mod H, (n+j-kc) mod W] (correlation)
// One block = one 32x32 output tile of one channel of one image; the input tile
// with its (ks-1)-wide periodic halo is staged in shared memory.
constexpr int BT = 32;

__device__ __forceinline__ int wrapi(int v, int n) { v %= n; return v < 0 ? v + n : v; }

template <bool ADJ>
__device__ __forceinline__ void blur_tile(const float* __restrict__ src, const float* __restrict__ kern,
                                          int ks, int H, int W, int m0, int n0, float* tile, float* ksm,
                                          float out[4]) {
  const int kc = (ks - 1) / 2;
  const int TW = BT + ks - 1;
  for (int t = threadIdx.x; t < ks * ks; t += blockDim.x) ksm[t] = kern[t];
  // tile[u][v] holds src[m0 - kc + u][n0 - kc + v] (periodic)
  for (int t = threadIdx.x; t < TW * TW; t += blockDim.x) {
    const int u = t / TW, v = t % TW;
    tile[t] = src[(long long)wrapi(m0 - kc + u, H) * W + wrapi(n0 - kc + v, W)];
  }
  __syncthreads();
  const int tx = threadIdx.x & 31, ty0 = threadIdx.x >> 5;  // 8 rows of threads x 4 rows each
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int ty = ty0 + 8 * q;
    float s = 0.f;
    for (int i = 0; i < ks; ++i) {
      for (int j = 0; j < ks; ++j) {
        // forward: x[m - i + kc]  -> tile row ty - i + 2kc ; adjoint: r[m + i - kc] -> tile row ty + i
        const int u = ADJ ? (ty + i) : (ty - i + 2 * kc);
        const int v = ADJ ? (tx + j) : (tx - j + 2 * kc);
        s = fmaf(ksm[i * ks + j], tile[u * TW + v], s);
      }
    }
    out[q] = s;
  }
}

// r = A z - y
__global__ void __launch_bounds__(256) blur_residual_kernel(StepArgs a) {
  pdl_enter();
  extern __shared__ float sm[];
  const int n = blockIdx.z / a.C, c = blockIdx.z % a.C;
  if (a.active && !a.active[n]) return;
  const int m0 = blockIdx.y * BT, n0 = blockIdx.x * BT;
  const long long plane = ((long long)n * a.C + c) * a.H * a.W;
  const float* kern = a.kern + (a.kernel_per_image ? (long long)n * a.ksize * a.ksize : 0);
  float* ksm = sm;
  float* tile = sm + a.ksize * a.ksize;
  float out[4];
  blur_tile<false>(a.z + plane, kern, a.ksize, a.H, a.W, m0, n0, tile, ksm, out);
  const int tx = threadIdx.x & 31, ty0 = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int m = m0 + ty0 + 8 * q, nn = n0 + tx;
    if (m < a.H && nn < a.W) {
      const long long i = plane + (long long)m * a.W + nn;
      a.fbuf[i] = out[q] - (a.y ? a.y[i] : 0.f);
    }
  }
}

// out = A^T src (used for A^T(Az - y) in the gradient step and A^T y for the prox)
// MODE 0: plain store into a.fbuf2 ; MODE 1: fused gradient step + tail.
template <int MODE>
__global__ void __launch_bounds__(256) blur_adjoint_kernel(StepArgs a, const float* __restrict__ src) {
  pdl_enter();
  extern __shared__ float sm[];
  const int n = blockIdx.z / a.C, c = blockIdx.z % a.C;
  if (a.active && !a.active[n]) return;
  const int m0 = blockIdx.y * BT, n0 = blockIdx.x * BT;
  const long long plane = ((long long)n * a.C + c) * a.H * a.W;
  const float* kern = a.kern + (a.kernel_per_image ? (long long)n * a.ksize * a.ksize : 0);
  float* ksm = sm;
  float* tile = sm + a.ksize * a.ksize;
  float out[4];
  blur_tile<true>(src + plane, kern, a.ksize, a.H, a.W, m0, n0, tile, ksm, out);
  const int tx = threadIdx.x & 31, ty0 = threadIdx.x >> 5;
  if (MODE == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int m = m0 + ty0 + 8 * q, nn = n0 + tx;
      if (m < a.H && nn < a.W) a.fbuf2[plane + (long long)m * a.W + nn] = out[q];
    }
    return;
  }
  const int k = *a.kdev;
  const float* xk_base = (k & 1) ? a.X1 : a.X0;
  float* xn_base = (k & 1) ? a.X0 : a.X1;
  Partial3 acc{0.f, 0.f, 0.f};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int m = m0 + ty0 + 8 * q, nn = n0 + tx;
    if (m < a.H && nn < a.W) {
      const long long i = plane + (long long)m * a.W + nn;
      // x^{k+1} = z - tau (A^T(Az - y) + lam grad g(z))   (Alg. 1 l.8)
      const float x1 = a.z[i] - a.tau * (out[q] + a.lam * a.gg[i]);
      tail_elem(x1, xk_base[i], a.beta, xn_base + i, a.zout + i, acc);
    }
  }
  const int tiles = gridDim.x * gridDim.y;
  const int part = c * tiles + blockIdx.y * gridDim.x + blockIdx.x;
  block_reduce_store(acc, a.partials + ((long long)n * a.parts + part) * 3);
}

// ---- register-blocked variant for the kernel sizes of the configs (KS = 9, 15, 25)
// One block = a 64 x 64 output tile of one channel plane, 128 threads; a thread owns 4 rows x 8
// consecutive columns. Per kernel row i it holds the row k[i][.] in registers (broadcast loads)
// and, per output row, the KS + 7 input values of its columns' window (float4 shared loads), so
// every value is reused for all 8 x KS products of that row: ~0.2 shared loads per FMA instead of
// the 2 of the one-output-per-thread loop above (which ran at ~9% of the FFMA peak, LSU-bound).
constexpr int BT2 = 64;
template <int KS>
struct Blur2 {
  static constexpr int KC = (KS - 1) / 2;
  static constexpr int TW = (BT2 + KS - 1 + 3) & ~3;  // tile row pitch (float4-aligned)
  static constexpr int SEG = (8 + KS - 1 + 3) & ~3;   // window registers per output row
  static constexpr size_t smem = sizeof(float) * (KS * KS + (size_t)(BT2 + KS - 1) * TW) + 16;
};
template <int KS, bool ADJ>
__device__ __forceinline__ void blur_tile2(const float* __restrict__ src, const float* __restrict__ kern, int H, int W,
                                           int m0, int n0, float* sm, float (&acc)[4][8]) {
  using B = Blur2<KS>;
  float* ksm = sm;
  float* tile = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(sm + KS * KS) + 15) & ~(uintptr_t)15);
  for (int t = threadIdx.x; t < KS * KS; t += blockDim.x) ksm[t] = kern[t];
  // tile[u][v] = src[m0 - kc + u][n0 - kc + v] (periodic), u, v < 64 + KS - 1
  constexpr int TH = BT2 + KS - 1;
  for (int t = threadIdx.x; t < TH * TH; t += blockDim.x) {
    const int u = t / TH, v = t - u * TH;
    tile[u * B::TW + v] = src[(long long)wrapi(m0 - B::KC + u, H) * W + wrapi(n0 - B::KC + v, W)];
  }
  __syncthreads();
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;  // 8 column groups x 16 row groups
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0.f;
#pragma unroll 1
  for (int i = 0; i < KS; ++i) {
    float kr[KS];
#pragma unroll
    for (int j = 0; j < KS; ++j) kr[j] = ksm[i * KS + j];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int y = ty * 4 + r;
      // forward: x[m - i + kc] -> tile row y - i + 2kc ; adjoint: r[m + i - kc] -> tile row y + i
      const int u = ADJ ? (y + i) : (y - i + 2 * B::KC);
      const float4* rowp = reinterpret_cast<const float4*>(tile + u * B::TW + tx * 8);
      float seg[B::SEG];
#pragma unroll
      for (int e = 0; e < B::SEG / 4; ++e) {
        const float4 q = rowp[e];
        seg[4 * e] = q.x; seg[4 * e + 1] = q.y; seg[4 * e + 2] = q.z; seg[4 * e + 3] = q.w;
      }
#pragma unroll
      for (int j = 0; j < KS; ++j)
#pragma unroll
        for (int c = 0; c < 8; ++c)
          // forward: tile col x - j + 2kc = (c + KS - 1 - j) in the window; adjoint: x + j = c + j
          acc[r][c] = fmaf(kr[j], seg[ADJ ? (c + j) : (c + KS - 1 - j)], acc[r][c]);
    }
  }
}

template <int KS>
__global__ void __launch_bounds__(128) blur_residual2_kernel(StepArgs a) {
  pdl_enter();
  extern __shared__ float sm[];
  const int n = blockIdx.z / a.C, c = blockIdx.z % a.C;
  if (a.active && !a.active[n]) return;
  const int m0 = blockIdx.y * BT2, n0 = blockIdx.x * BT2;
  const long long plane = ((long long)n * a.C + c) * a.H * a.W;
  const float* kern = a.kern + (a.kernel_per_image ? (long long)n * KS * KS : 0);
  float acc[4][8];
  blur_tile2<KS, false>(a.z + plane, kern, a.H, a.W, m0, n0, sm, acc);
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int m = m0 + ty * 4 + r;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int nn = n0 + tx * 8 + q;
      if (m < a.H && nn < a.W) {
        const long long i = plane + (long long)m * a.W + nn;
        a.fbuf[i] = acc[r][q] - (a.y ? a.y[i] : 0.f);
      }
    }
  }
}

template <int KS, int MODE>
__global__ void __launch_bounds__(128) blur_adjoint2_kernel(StepArgs a, const float* __restrict__ src) {
  pdl_enter();
  extern __shared__ float sm[];
  const int n = blockIdx.z / a.C, c = blockIdx.z % a.C;
  if (a.active && !a.active[n]) return;
  const int m0 = blockIdx.y * BT2, n0 = blockIdx.x * BT2;
  const long long plane = ((long long)n * a.C + c) * a.H * a.W;
  const float* kern = a.kern + (a.kernel_per_image ? (long long)n * KS * KS : 0);
  float acc[4][8];
  blur_tile2<KS, true>(src + plane, kern, a.H, a.W, m0, n0, sm, acc);
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;
  if (MODE == 0) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int m = m0 + ty * 4 + r;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int nn = n0 + tx * 8 + q;
        if (m < a.H && nn < a.W) a.fbuf2[plane + (long long)m * a.W + nn] = acc[r][q];
      }
    }
    return;
  }
  const int k = *a.kdev;
  const float* xk_base = (k & 1) ? a.X1 : a.X0;
  float* xn_base = (k & 1) ? a.X0 : a.X1;
  Partial3 pacc{0.f, 0.f, 0.f};
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int m = m0 + ty * 4 + r;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int nn = n0 + tx * 8 + q;
      if (m < a.H && nn < a.W) {
        const long long i = plane + (long long)m * a.W + nn;
        // x^{k+1} = z - tau (A^T(Az - y) + lam grad g(z))   (Alg. 1 l.8)
        const float x1 = a.z[i] - a.tau * (acc[r][q] + a.lam * a.gg[i]);
        tail_elem(x1, xk_base[i], a.beta, xn_base + i, a.zout + i, pacc);
      }
    }
  }
  const int tiles = gridDim.x * gridDim.y;
  const int part = c * tiles + blockIdx.y * gridDim.x + blockIdx.x;
  block_reduce_store(pacc, a.partials + ((long long)n * a.parts + part) * 3);
}

static bool blur2_ks(int ks) { return ks == 9 || ks == 15 || ks == 25; }
// the register-blocked kernel needs whole 64 x 64 tiles to pay off; smaller planes (C1's 32 x 32)
// keep the 32 x 32-tile kernel (a 64-tile block would leave 3/4 of its threads' outputs idle)
static bool use_blur2(int ks, int H, int W) { return blur2_ks(ks) && H >= BT2 && W >= BT2; }

// ------------------------------------------------------------------ finalize / stop logic
// One warp per image: fixed-order fp64 combine of the partials, r = sqrt(d2)/sqrt(n2),
// divergence (any non-finite x^{k+1}: keep x^k, reading Q22) and the per-image stop
// rule at check iterations (reading Q17).
__global__ void finalize_kernel(FinalizeArgs f) {
  pdl_enter();
  const int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (n >= f.N) return;
  if (!f.active[n]) {
    if (lane == 0) { f.r_now[n] = __int_as_float(0x7fc00000); if (f.flags) f.flags[n] = 0; }
    return;
  }
  const int k = *f.kdev;
  double d2 = 0.0, n2 = 0.0, bad = 0.0;
  for (int p = lane; p < f.parts; p += 32) {
    const float* q = f.partials + ((long long)n * f.parts + p) * 3;
    d2 += (double)q[0]; n2 += (double)q[1]; bad += (double)q[2];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    d2 += __shfl_xor_sync(0xffffffffu, d2, o);
    n2 += __shfl_xor_sync(0xffffffffu, n2, o);
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if (lane != 0) return;
  if (bad > 0.0 || !isfinite(d2)) {
    f.status[n] = 2;
    f.active[n] = 0;
    f.r_now[n] = __int_as_float(0x7fc00000);
    if (f.flags) f.flags[n] = 0;
    return;
  }
  if (f.flags) {  // NEXT-1 bookkeeping of the accepted step (fp64, like the oracle)
    int fl = 1;
    if (f.restart) {  // Eq. 5: k * sum_{t<k} ||x^{t+1} - x^t||^2 > B^2
      int kr = f.rk[n] + 1;
      double S = f.rsum[n] + d2;
      if ((double)kr * S > f.B2) {
        fl |= 2;
        f.nrest[n] += 1;
        if (f.restart == 1) { kr = 0; S = 0.0; }  // Alg. 1: k <- 0; Alg. 2 keeps both
      }
      f.rk[n] = kr;
      f.rsum[n] = S;
    }
    if (f.averaging && k > f.K / 2 && k < f.K - 1) {  // window floor(K/2) < k < K-1
      const float inc = (float)sqrt(d2);
      if (inc < f.best[n]) { f.best[n] = inc; f.k0[n] = k; fl |= 4; }  // strict: first minimum
    }
    f.flags[n] = fl;
  }
  const double r = n2 > 0.0 ? sqrt(d2) / sqrt(n2) : (double)INFINITY;
  f.iters[n] = k + 1;
  f.res[n] = (float)r;
  f.r_now[n] = (float)r;
  if (f.stop_rule == 0 && ((k + 1) % f.check_every) == 0 && (float)r <= f.tol) {
    f.active[n] = 0;
    f.status[n] = 0;
  }
}

// Single block: max over the images updated in this iteration (trace), the local
// max for the global rule (all-reduced between the two phases when world > 1),
// then the global-max decision, the active count the host polls, and k += 1.
__global__ void advance_a_kernel(FinalizeArgs f) {
  pdl_enter();
  __shared__ float smax[32];
  float m = -1.f;
  for (int n = threadIdx.x; n < f.N; n += blockDim.x) {
    const float r = f.r_now[n];
    if (!isnan(r)) m = fmaxf(m, r);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) smax[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, smax[w]);
    m = fmaxf(m, smax[0]);
    const int k = *f.kdev;
    if (f.trace && k < f.trace_cap) f.trace[k] = m >= 0.f ? m : __int_as_float(0x7fc00000);
    *f.rmax = m;  // -1 = no image updated on this rank
  }
}

__global__ void advance_b_kernel(FinalizeArgs f) {
  pdl_enter();
  __shared__ int cnt[32];
  __shared__ int stop_all;
  const int k = *f.kdev;
  if (threadIdx.x == 0) {
    const float m = *f.rmax;  // global max after the all-reduce (or local when world == 1)
    stop_all = (f.stop_rule == 1 && ((k + 1) % f.check_every) == 0 && m >= 0.f && m <= f.tol);
  }
  __syncthreads();
  int c = 0;
  for (int n = threadIdx.x; n < f.N; n += blockDim.x) {
    if (f.active[n]) {
      if (stop_all) { f.active[n] = 0; f.status[n] = 0; } else { ++c; }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) cnt[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += cnt[w];
    *f.n_active = s;
    *f.kdev = k + 1;
  }
  // compacted list of the active images in index order (the conv kernels' live tiles), built in
  // chunks of blockDim.x images: a ballot per warp, a prefix over the warps of the chunk, and a
  // running offset carried from chunk to chunk (any N)
  if (f.act_list) {
    __shared__ int run;
    __syncthreads();  // thread 0 has read the counts in cnt[] before they are overwritten
    if (threadIdx.x == 0) run = 0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int base = 0; base < f.N; base += blockDim.x) {
      const int n = base + threadIdx.x;
      const int a = (n < f.N && f.active[n]) ? 1 : 0;
      const unsigned bal = __ballot_sync(0xffffffffu, a);
      if (lane == 0) cnt[w] = __popc(bal);
      __syncthreads();
      int off = run;
      for (int i = 0; i < w; ++i) off += cnt[i];
      if (a) f.act_list[off + __popc(bal & ((1u << lane) - 1u))] = n;
      __syncthreads();  // every thread has read run and cnt[]
      if (threadIdx.x == 0) {
        int s = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += cnt[i];
        run += s;
      }
      __syncthreads();
    }
  }
}

// x-hat_n = x^{iters_n}: images whose last accepted iterate sits in X1 are copied to X0.
__global__ void gather_kernel(const int* __restrict__ iters, const float* __restrict__ X1, float* __restrict__ X0,
                              long long d) {
  const int n = blockIdx.y;
  if ((iters[n] & 1) == 0) return;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < d; e += (long long)gridDim.x * blockDim.x)
    X0[(long long)n * d + e] = X1[(long long)n * d + e];
}

// After finalize, per image that stepped: restart -> z^{k+1} := x^{k+1} (the inertia reset of
// Eq. 5 / Alg. 1 l.10 / Alg. 2 l.10); averaging -> snapshot mean(z^0..z^k) on a new window
// minimum, then add z^{k+1} to the running sum (O(1) planes instead of the whole trajectory).
__global__ void __launch_bounds__(256) post_step_kernel(PostArgs a) {
  pdl_enter();
  const int n = blockIdx.y;
  const int fl = a.flags[n];
  if (!(fl & 1)) return;
  const bool rs = (fl & 2) != 0, snap = (fl & 4) != 0;
  if (!rs && !a.Zsum) return;
  const int k = *a.kdev;
  const float* xn = ((k & 1) ? a.X0 : a.X1) + (long long)n * a.d;
  float* z = a.Z + (long long)n * a.d;
  const float inv = 1.f / (float)(k + 1);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < a.d; e += (long long)gridDim.x * blockDim.x) {
    float z1 = z[e];
    if (rs) { z1 = xn[e]; z[e] = z1; }
    if (a.Zsum) {
      float* zs = a.Zsum + (long long)n * a.d;
      const float sum = zs[e];
      if (snap) a.Xsnap[(long long)n * a.d + e] = sum * inv;
      zs[e] = sum + z1;
    }
  }
}

void launch_post_step(const PostArgs& a, cudaStream_t s) {
  const long long bx = (a.d + 256 * 8 - 1) / (256 * 8);
  launch_k(post_step_kernel, dim3((unsigned)(bx < 1 ? 1 : bx), a.N), 256, 0, s, a);
}

// x-hat = the averaging snapshot for images with a K0 (not diverged)
__global__ void avg_out_kernel(const int* __restrict__ k0, const int* __restrict__ status,
                               const int* __restrict__ iters, int K, const float* __restrict__ Xsnap,
                               float* __restrict__ X, long long d) {
  const int n = blockIdx.y;
  if (k0[n] < 0 || status[n] == 2 || iters[n] != K) return;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < d; e += (long long)gridDim.x * blockDim.x)
    X[(long long)n * d + e] = Xsnap[(long long)n * d + e];
}

void launch_avg_out(const int* k0, const int* status, const int* iters, int K, const float* Xsnap, float* X, int N,
                    long long d, cudaStream_t s) {
  const long long bx = (d + 256 * 8 - 1) / (256 * 8);
  avg_out_kernel<<<dim3((unsigned)(bx < 1 ? 1 : bx), N), 256, 0, s>>>(k0, status, iters, K, Xsnap, X, d);
}

__global__ void init_state_kernel(FinalizeArgs f) {
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < f.N; n += gridDim.x * blockDim.x) {
    f.active[n] = 1;
    if (f.act_list) f.act_list[n] = n;
    f.status[n] = 1;
    f.iters[n] = 0;
    f.res[n] = __int_as_float(0x7fc00000);
    f.r_now[n] = __int_as_float(0x7fc00000);
    if (f.flags) {
      f.flags[n] = 0;
      f.rk[n] = 0;
      f.rsum[n] = 0.0;
      f.nrest[n] = 0;
      f.best[n] = __int_as_float(0x7f800000);
      f.k0[n] = -1;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) { *f.kdev = 0; *f.n_active = f.N; }
}

// Elementwise helpers for the component entry points.
__global__ void inpaint_grad_kernel(const float* __restrict__ x, const float* __restrict__ y,
                                    const uint8_t* __restrict__ mask, float* __restrict__ out,
                                    long long total, long long HW, long long CHW) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const float m = (float)mask[(i / CHW) * HW + (i % HW)];
    out[i] = m * (m * x[i] - y[i]);
  }
}

__global__ void inpaint_prox_kernel(const float* __restrict__ v, const float* __restrict__ y,
                                    const uint8_t* __restrict__ mask, float tau, float* __restrict__ out,
                                    long long total, long long HW, long long CHW) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const float m = (float)mask[(i / CHW) * HW + (i % HW)];
    out[i] = (tau * m * y[i] + v[i]) / (tau * m + 1.f);
  }
}

// ------------------------------------------------------------------ launchers
void launch_pointwise_step(int mode, const StepArgs& a, cudaStream_t s) {
  dim3 grid(a.parts, a.N);
  if (a.d % 4 == 0 && ((long long)a.H * a.W) % 4 == 0) {
    switch (mode) {
      case STEP_PROX_INPAINT: launch_k(pointwise_step_v4_kernel<STEP_PROX_INPAINT>, grid, 256, 0, s, a); return;
      case STEP_GRAD_BUF: launch_k(pointwise_step_v4_kernel<STEP_GRAD_BUF>, grid, 256, 0, s, a); return;
      case STEP_GRAD_INPAINT: launch_k(pointwise_step_v4_kernel<STEP_GRAD_INPAINT>, grid, 256, 0, s, a); return;
      case STEP_GRAD_RICIAN: launch_k(pointwise_step_v4_kernel<STEP_GRAD_RICIAN>, grid, 256, 0, s, a); return;
      case STEP_GRAD_MRI: launch_k(pointwise_step_v4_kernel<STEP_GRAD_MRI>, grid, 256, 0, s, a); return;
      default: launch_k(pointwise_step_v4_kernel<STEP_X1_BUF>, grid, 256, 0, s, a); return;
    }
  }
  switch (mode) {
    case STEP_PROX_INPAINT: launch_k(pointwise_step_kernel<STEP_PROX_INPAINT>, grid, 256, 0, s, a); break;
    case STEP_GRAD_BUF: launch_k(pointwise_step_kernel<STEP_GRAD_BUF>, grid, 256, 0, s, a); break;
    case STEP_GRAD_INPAINT: launch_k(pointwise_step_kernel<STEP_GRAD_INPAINT>, grid, 256, 0, s, a); break;
    case STEP_GRAD_RICIAN: launch_k(pointwise_step_kernel<STEP_GRAD_RICIAN>, grid, 256, 0, s, a); break;
    case STEP_GRAD_MRI: launch_k(pointwise_step_kernel<STEP_GRAD_MRI>, grid, 256, 0, s, a); break;
    default: launch_k(pointwise_step_kernel<STEP_X1_BUF>, grid, 256, 0, s, a); break;
  }
}

static size_t blur_smem(int ks) { return sizeof(float) * (ks * ks + (BT + ks - 1) * (BT + ks - 1)); }

int blur_parts_per_image(int C, int H, int W, int ks) {
  const int bt = use_blur2(ks, H, W) ? BT2 : BT;
  return C * ((H + bt - 1) / bt) * ((W + bt - 1) / bt);
}

template <int KS>
static void launch_blur2(int which, const StepArgs& a, const float* src, cudaStream_t s) {
  dim3 grid((a.W + BT2 - 1) / BT2, (a.H + BT2 - 1) / BT2, a.N * a.C);
  const size_t sm = Blur2<KS>::smem;
  if (which == 0) launch_k(blur_residual2_kernel<KS>, grid, 128, sm, s, a);
  else if (which == 1) launch_k(blur_adjoint2_kernel<KS, 0>, grid, 128, sm, s, a, src);
  else launch_k(blur_adjoint2_kernel<KS, 1>, grid, 128, sm, s, a, src);
}
static bool launch_blur2_any(int which, const StepArgs& a, const float* src, cudaStream_t s) {
  if (!use_blur2(a.ksize, a.H, a.W)) return false;
  switch (a.ksize) {
    case 9: launch_blur2<9>(which, a, src, s); return true;
    case 15: launch_blur2<15>(which, a, src, s); return true;
    case 25: launch_blur2<25>(which, a, src, s); return true;
    default: return false;
  }
}

void launch_blur_residual(const StepArgs& a, cudaStream_t s) {
  if (launch_blur2_any(0, a, nullptr, s)) return;
  dim3 grid((a.W + BT - 1) / BT, (a.H + BT - 1) / BT, a.N * a.C);
  const size_t sm = blur_smem(a.ksize);
  launch_k(blur_residual_kernel, grid, 256, sm, s, a);
}

void launch_blur_adjoint(int mode, const StepArgs& a, const float* src, cudaStream_t s) {
  if (launch_blur2_any(mode == 0 ? 1 : 2, a, src, s)) return;
  dim3 grid((a.W + BT - 1) / BT, (a.H + BT - 1) / BT, a.N * a.C);
  const size_t sm = blur_smem(a.ksize);
  if (mode == 0) {
    launch_k(blur_adjoint_kernel<0>, grid, 256, sm, s, a, src);
  } else {
    launch_k(blur_adjoint_kernel<1>, grid, 256, sm, s, a, src);
  }
}

void init_attrs_step() {

  set_max_dyn_smem(blur_residual_kernel);
  set_max_dyn_smem(blur_adjoint_kernel<0>);
  set_max_dyn_smem(blur_adjoint_kernel<1>);
  set_max_dyn_smem(blur_residual2_kernel<25>);
  set_max_dyn_smem(blur_adjoint2_kernel<25, 0>);
  set_max_dyn_smem(blur_adjoint2_kernel<25, 1>);
}

void launch_finalize(const FinalizeArgs& f, cudaStream_t s) {
  launch_k(finalize_kernel, (f.N + 7) / 8, 256, 0, s, f);
}
void launch_advance_a(const FinalizeArgs& f, cudaStream_t s) { launch_k(advance_a_kernel, 1, 1024, 0, s, f); }
void launch_advance_b(const FinalizeArgs& f, cudaStream_t s) { launch_k(advance_b_kernel, 1, 1024, 0, s, f); }
void launch_init_state(const FinalizeArgs& f, cudaStream_t s) { init_state_kernel<<<(f.N + 255) / 256, 256, 0, s>>>(f); }
void launch_gather(const int* iters, const float* X1, float* X0, int N, long long d, cudaStream_t s) {
  dim3 grid((unsigned)std::min<long long>((d + 255) / 256, 1024), N);
  gather_kernel<<<grid, 256, 0, s>>>(iters, X1, X0, d);
}
void launch_inpaint_grad(const float* x, const float* y, const uint8_t* m, float* out, int N, int C, int H, int W,
                         cudaStream_t s) {
  const long long total = (long long)N * C * H * W;
  inpaint_grad_kernel<<<(unsigned)std::min<long long>((total + 255) / 256, 65535), 256, 0, s>>>(
      x, y, m, out, total, (long long)H * W, (long long)C * H * W);
}
void launch_inpaint_prox(const float* v, const float* y, const uint8_t* m, float tau, float* out, int N, int C, int H,
                         int W, cudaStream_t s) {
  const long long total = (long long)N * C * H * W;
  inpaint_prox_kernel<<<(unsigned)std::min<long long>((total + 255) / 256, 65535), 256, 0, s>>>(
      v, y, m, tau, out, total, (long long)H * W, (long long)C * H * W);
}

}  // namespace ideq

namespace ideq {
// Off: on B200 the programmatic launch of the small per-iteration kernels (and of the fused head)
// measured ~1% SLOWER on the C3 bench (10.20k vs 10.32k img-it/s, 3 interleaved A/B pairs) and no
// better on the latency-bound C1 -- the early-launched CTAs wait in SM slots while the persistent
// conv grids run. The kernels call griddepcontrol.wait either way (a no-op without the attribute);
// building with -DIDEQ_PDL_SMALL=1 turns the attribute on.
#ifndef IDEQ_PDL_SMALL
#define IDEQ_PDL_SMALL 0
#endif
bool pdl_enabled() { return IDEQ_PDL_SMALL != 0; }
}  // namespace ideq
