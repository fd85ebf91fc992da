// Hand-written batched 2-D FFTs for the fidelity operators that need them:
//
//  * periodic blur prox (BASELINE C5): x = F^-1[ F(v + tau A^T y) / (1 + tau |K^|^2) ]
//    (I + tau A^T A is circulant, so the prox is a diagonal solve in Fourier space;
//    the DFT normalisation cancels). Real planes -> half spectrum [H][W/2+1].
//  * coded-diffraction phase retrieval (BASELINE C4), unitary F:
//    grad f = sum_j 2 Re( conj(D_j) F^-1[ (|u_j|^2 - y_j) u_j ] ),  u_j = F(D_j z).
//
// Each 2-D transform is a row pass (contiguous rows, one or more rows per block) and
// a column pass (a block owns a strip of columns), each an in-shared-memory radix-2
// FFT with fp32 twiddles computed in fp64 on the host. The pointwise work (prox
// right-hand side, diagonal solve, phase residual, conj(D_j) combine) and the final
// update + residual partials are fused into the passes, so every plane crosses HBM a
// fixed small number of times. Sizes are powers of two up to 1024.
#include "common.cuh"
#include "kernels.h"

namespace ideq {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cconjmul(float2 a, float2 b) {  // conj(a) * b
  return make_float2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}

// Shared-memory rows are padded by one float2 per 16 (pd): the bit-reversed scatter of a row
// (consecutive i -> indices N/32 apart) and the short-stride butterflies of the first passes
// otherwise fall on 1-2 bank groups (up to 16-way conflicts). Column buffers additionally get an
// odd pitch so the FFT_CPB columns a warp loads row by row land on different banks.
__host__ __device__ __forceinline__ int pd(int i) { return i + (i >> 4); }
__host__ __device__ __forceinline__ int row_pitch(int N) { return N + N / 16; }
__host__ __device__ __forceinline__ int col_pitch(int N) { return N + N / 16 + 1; }

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }

// In-place DIT FFT of one length-N row held in shared memory in BIT-REVERSED order. `t` is this
// thread's index among the `tpr` threads that own the row. Every thread of the block must call
// this (it synchronises the block between passes). tw[k] = exp(-2 pi i k / N), k < N/2.
// inverse = unnormalised inverse transform. The radix-2 stages are fused in pairs (radix-4
// passes: each thread combines 4 points in registers through both stages), so a 256-point row
// takes 4 shared-memory round trips and barriers instead of 8; an odd log N starts with one
// radix-2 pass.
__device__ __forceinline__ void fft_row(float2* d, const float2* tw, int N, int logN, int t, int tpr, bool inverse) {
  int s = 1;
  if (logN & 1) {  // stage 1: pairs (2b, 2b + 1), twiddle 1
    for (int b = t; b < (N >> 1); b += tpr) {
      const float2 a = d[pd(2 * b)], c = d[pd(2 * b + 1)];
      d[pd(2 * b)] = cadd(a, c);
      d[pd(2 * b + 1)] = csub(a, c);
    }
    __syncthreads();
    s = 2;
  }
  for (; s < logN; s += 2) {  // stages s and s + 1
    const int h = 1 << (s - 1);
    const int step1 = N >> s, step2 = N >> (s + 1);
    for (int b = t; b < (N >> 2); b += tpr) {
      const int j = b & (h - 1);
      const int i0 = ((b >> (s - 1)) << (s + 1)) + j;
      float2 w1 = tw[j * step1], w2 = tw[j * step2], w3 = tw[(j + h) * step2];
      if (inverse) { w1.y = -w1.y; w2.y = -w2.y; w3.y = -w3.y; }
      const int p0 = pd(i0), p1 = pd(i0 + h), p2 = pd(i0 + 2 * h), p3 = pd(i0 + 3 * h);
      const float2 x0 = d[p0], x1 = d[p1], x2 = d[p2], x3 = d[p3];
      // stage s: butterflies (i0, i0 + h) and (i0 + 2h, i0 + 3h), both at offset j of their 2h block
      const float2 t1 = cmul(w1, x1), t3 = cmul(w1, x3);
      const float2 a0 = cadd(x0, t1), a1 = csub(x0, t1), b0 = cadd(x2, t3), b1 = csub(x2, t3);
      // stage s + 1: butterflies (i0, i0 + 2h) at offset j and (i0 + h, i0 + 3h) at offset j + h
      const float2 u2 = cmul(w2, b0), u3 = cmul(w3, b1);
      d[p0] = cadd(a0, u2);
      d[p2] = csub(a0, u2);
      d[p1] = cadd(a1, u3);
      d[p3] = csub(a1, u3);
    }
    __syncthreads();
  }
}

__host__ __device__ __forceinline__ int fft_tpr(int W) { return (W / 4) < 32 ? (W / 4 > 0 ? W / 4 : 1) : 32; }

__device__ __forceinline__ int bitrev(int i, int logN) { return (int)(__brev((unsigned)i) >> (32 - logN)); }

// natural -> bit-reversed order in place (the owner of the smaller index swaps each pair), then a
// block barrier
__device__ __forceinline__ void bitrev_permute(float2* d, int N, int logN, int t, int tpr) {
  for (int i = t; i < N; i += tpr) {
    const int r = bitrev(i, logN);
    if (i < r) {
      const float2 a = d[pd(i)];
      d[pd(i)] = d[pd(r)];
      d[pd(r)] = a;
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void load_twiddles(float2* s_tw, const float2* g_tw, int N) {
  for (int k = threadIdx.x; k < N / 2; k += blockDim.x) s_tw[k] = g_tw[k];
}

// ------------------------------------------------------------------ shared tail (update + partials)
struct P3 { float d2, n2, bad; };

__device__ __forceinline__ void reduce_store_p3(P3 v, float* out3) {
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
    P3 s{lane < nw ? red[0][lane] : 0.f, lane < nw ? red[1][lane] : 0.f, lane < nw ? red[2][lane] : 0.f};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s.d2 += __shfl_xor_sync(0xffffffffu, s.d2, o);
      s.n2 += __shfl_xor_sync(0xffffffffu, s.n2, o);
      s.bad += __shfl_xor_sync(0xffffffffu, s.bad, o);
    }
    if (lane == 0) { out3[0] = s.d2; out3[1] = s.n2; out3[2] = s.bad; }
  }
}

__device__ __forceinline__ void step_tail(float x1, long long i, const StepArgs& a, const float* xk_base,
                                          float* xn_base, P3& acc) {
  const float xk = xk_base[i];
  xn_base[i] = x1;
  a.zout[i] = x1 + a.beta * (x1 - xk);
  const float d = x1 - xk;
  if (isfinite(x1)) acc.d2 += d * d; else acc.bad += 1.f;
  acc.n2 += xk * xk;
}

// ================================================================== blur (real planes)
// Row pass, forward: one real row -> W-point complex FFT -> half spectrum (W/2+1).
//   mode 0: input = src plane
//   mode 1: input = v + tau A^T y = z - tau lam grad g + tau ATy   (prox right-hand side)
__global__ void __launch_bounds__(256) blur_rows_fwd_kernel(FftArgs f, const float* __restrict__ src, int mode) {
  pdl_enter();
  extern __shared__ float2 sm2[];
  const int W = f.W, logW = f.logW;
  const int tpr = fft_tpr(W);
  const int rpb = 256 / tpr;
  float2* tw = sm2;
  float2* rows = sm2 + W / 2;
  load_twiddles(tw, f.tw_w, W);
  const int r = threadIdx.x / tpr, t = threadIdx.x % tpr;
  const int h = blockIdx.x * rpb + r;
  const int c = blockIdx.y, n = blockIdx.z;
  if (f.active && !f.active[n]) return;  // uniform per block
  float2* d = rows + r * row_pitch(W);
  const long long plane = ((long long)n * f.C + c) * f.H * W;
  if (h < f.H) {
    for (int i = t; i < W; i += tpr) {
      const long long e = plane + (long long)h * W + i;
      float v;
      if (mode == 1) v = f.z[e] - f.tau * f.lam * f.gg[e] + f.tau * f.aty[e];
      else v = src[e];
      d[pd(bitrev(i, logW))] = make_float2(v, 0.f);
    }
  }
  __syncthreads();
  fft_row(d, tw, W, logW, t, tpr, false);
  if (h < f.H) {
    const int Wh = W / 2 + 1;
    float2* S = f.spec + ((long long)n * f.C + c) * f.H * Wh + (long long)h * Wh;
    for (int i = t; i < Wh; i += tpr) S[i] = d[pd(i)];
  }
}

// Column pass on the half spectrum: forward H-point FFT, pointwise op, inverse FFT.
//   op 0: multiply by the real diagonal dgl[ky][kx] = 1 / (1 + tau |K^|^2)   (prox)
//   op 1: multiply by conj(K^[ky][kx])                                     (A^T)
//   op 2: forward only (no inverse): used to build K^ itself
//   op 3: inverse only (the half spectrum is already in k-space: MRI A^T y)
// Columns per block in column passes (16 threads per column) and threads per row in row passes
// (32, so a 256-thread block transforms 8 rows of 256 points): enough independent transforms per
// block to amortise the twiddle load and the per-pass barriers (2 rows / 8 columns per block ran
// the C4 passes at ~0.5 TB/s).
constexpr int FFT_CPB = 16;

__global__ void __launch_bounds__(256) blur_cols_kernel(FftArgs f, int op) {
  pdl_enter();
  extern __shared__ float2 sm2[];
  const int H = f.H, logH = f.logH;
  const int Wh = f.W / 2 + 1;
  float2* tw = sm2;
  float2* cols = sm2 + H / 2;
  load_twiddles(tw, f.tw_h, H);
  const int tpc = 256 / FFT_CPB;
  const int cc = threadIdx.x / tpc, t = threadIdx.x % tpc;
  const int kx0 = blockIdx.x * FFT_CPB;
  const int c = blockIdx.y, n = blockIdx.z;
  if (f.active && !f.active[n]) return;
  float2* S = f.spec + ((long long)n * f.C + c) * H * Wh;
  // coalesced-ish load: consecutive threads walk the FFT_CPB columns of a row
  for (int q = threadIdx.x; q < H * FFT_CPB; q += blockDim.x) {
    const int h = q / FFT_CPB, j = q % FFT_CPB;
    const int kx = kx0 + j;
    cols[j * col_pitch(H) + pd(bitrev(h, logH))] = kx < Wh ? S[(long long)h * Wh + kx] : make_float2(0.f, 0.f);
  }
  __syncthreads();
  float2* d = cols + cc * col_pitch(H);
  const int kx = kx0 + cc;
  if (op == 3) {  // loaded bit-reversed: straight into the inverse transform
    fft_row(d, tw, H, logH, t, tpc, true);
    for (int q = threadIdx.x; q < H * FFT_CPB; q += blockDim.x) {
      const int h = q / FFT_CPB, j = q % FFT_CPB;
      if (kx0 + j < Wh) S[(long long)h * Wh + kx0 + j] = cols[j * col_pitch(H) + pd(h)];
    }
    return;
  }
  fft_row(d, tw, H, logH, t, tpc, false);
  if (op == 2) {
    for (int q = threadIdx.x; q < H * FFT_CPB; q += blockDim.x) {
      const int h = q / FFT_CPB, j = q % FFT_CPB;
      if (kx0 + j < Wh) S[(long long)h * Wh + kx0 + j] = cols[j * col_pitch(H) + pd(h)];
    }
    return;
  }
  // pointwise op in natural order (in place), then the bit-reversal permutation for the inverse
  // pass (pairwise swaps; fft_row ended with a barrier)
  for (int ky = t; ky < H; ky += tpc) {
    float2 v = d[pd(ky)];
    if (kx < Wh) {
      if (op == 0) {
        const float g = f.dgl[(long long)ky * Wh + kx];
        v.x *= g; v.y *= g;
      } else {
        v = cconjmul(f.khat[(long long)ky * Wh + kx], v);
      }
    }
    d[pd(ky)] = v;
  }
  __syncthreads();
  bitrev_permute(d, H, logH, t, tpc);
  fft_row(d, tw, H, logH, t, tpc, true);
  for (int q = threadIdx.x; q < H * FFT_CPB; q += blockDim.x) {
    const int h = q / FFT_CPB, j = q % FFT_CPB;
    if (kx0 + j < Wh) S[(long long)h * Wh + kx0 + j] = cols[j * col_pitch(H) + pd(h)];
  }
}

// Row pass, inverse: half spectrum -> Hermitian full row -> inverse FFT -> real / (H W).
//   mode 0: store into dst plane ; mode 1: x^{k+1} -> update + residual partials.
__global__ void __launch_bounds__(256) blur_rows_inv_kernel(FftArgs f, StepArgs a, float* __restrict__ dst, int mode) {
  pdl_enter();
  extern __shared__ float2 sm2[];
  const int W = f.W, logW = f.logW, H = f.H;
  const int tpr = fft_tpr(W);
  const int rpb = 256 / tpr;
  float2* tw = sm2;
  float2* rows = sm2 + W / 2;
  load_twiddles(tw, f.tw_w, W);
  const int r = threadIdx.x / tpr, t = threadIdx.x % tpr;
  const int h = blockIdx.x * rpb + r;
  const int c = blockIdx.y, n = blockIdx.z;
  if (f.active && !f.active[n]) return;
  float2* d = rows + r * row_pitch(W);
  const int Wh = W / 2 + 1;
  if (h < H) {
    const float2* S = f.spec + ((long long)n * f.C + c) * H * Wh + (long long)h * Wh;
    for (int i = t; i < W; i += tpr) {
      float2 v = i < Wh ? S[i] : S[W - i];
      if (i >= Wh) v.y = -v.y;  // X[W-k] = conj(X[k]) for a real row (per column transform keeps it)
      d[pd(bitrev(i, logW))] = v;
    }
  }
  __syncthreads();
  fft_row(d, tw, W, logW, t, tpr, true);
  const float scale = 1.f / ((float)H * (float)W);
  const long long plane = ((long long)n * f.C + c) * H * W;
  if (mode == 0) {
    if (h < H)
      for (int i = t; i < W; i += tpr) dst[plane + (long long)h * W + i] = d[pd(i)].x * scale;
    return;
  }
  const int k = *a.kdev;
  const float* xk_base = (k & 1) ? a.X1 : a.X0;
  float* xn_base = (k & 1) ? a.X0 : a.X1;
  P3 acc{0.f, 0.f, 0.f};
  if (h < H)
    for (int i = t; i < W; i += tpr) step_tail(d[pd(i)].x * scale, plane + (long long)h * W + i, a, xk_base, xn_base, acc);
  const int part = c * gridDim.x + blockIdx.x;
  reduce_store_p3(acc, a.partials + ((long long)n * a.parts + part) * 3);
}

// Note on the Hermitian expansion above: the column pass transforms each column kx of
// the row spectra independently, so after the forward 2-D pass the stored half plane
// is X[ky][kx], kx <= W/2. For the inverse row pass of row ky we need X'[ky][kx] for
// all kx of the *column-inverted* data, which is the row spectrum of a real row, hence
// Hermitian in kx: X'[ky][W-kx] = conj(X'[ky][kx]).

// ================================================================== MRI (App. D.3.1)
// Half spectrum of the Hermitian part of M y, scaled: spec[ky][kx] = scale * M[ky][kx] *
// (y[ky][kx] + conj(y[-ky][-kx])) / 2, kx <= W/2. With a Hermitian-symmetric mask, the real part
// of F^-1(M y) is F^-1 of this Hermitian array (reading R7), i.e. a C2R transform of the half plane.
__global__ void mri_fill_kernel(const float* __restrict__ y, const uint8_t* __restrict__ kmask, float2* __restrict__ spec,
                                int H, int W, float scale) {
  const int Wh = W / 2 + 1;
  const int n = blockIdx.y;
  const float2* yc = reinterpret_cast<const float2*>(y) + (long long)n * H * W;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < H * Wh; e += gridDim.x * blockDim.x) {
    const int ky = e / Wh, kx = e % Wh;
    const float m = (float)kmask[ky * W + kx];
    const float2 a = yc[ky * W + kx];
    const float2 b = yc[((H - ky) % H) * W + (W - kx) % W];
    spec[(long long)n * H * Wh + e] = make_float2(0.5f * scale * m * (a.x + b.x), 0.5f * scale * m * (a.y - b.y));
  }
}
// mhalf = M on the half plane (gradient pass), dgl = 1 / (1 + tau M) (prox pass)
__global__ void mri_masks_kernel(const uint8_t* __restrict__ kmask, float* __restrict__ mhalf, float* __restrict__ dgl,
                                 float tau, int H, int W) {
  const int Wh = W / 2 + 1;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < H * Wh; e += gridDim.x * blockDim.x) {
    const float m = (float)kmask[(e / Wh) * W + e % Wh];
    mhalf[e] = m;
    dgl[e] = 1.f / (1.f + tau * m);
  }
}

// Embed the kernel: plane[(i-kc) mod H][(j-kc) mod W] = k[i][j] (tap (kc,kc) at the origin).
// The runtime requires ksize <= min(H, W), so no two taps share a bin.
__global__ void embed_kernel_kernel(const float* __restrict__ k, int ks, float* __restrict__ plane, int H, int W) {
  const int kc = (ks - 1) / 2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ks * ks; e += gridDim.x * blockDim.x) {
    const int i = e / ks, j = e % ks;
    const int r = ((i - kc) % H + H) % H, s = ((j - kc) % W + W) % W;
    plane[r * W + s] = k[e];
  }
}

// dgl = 1 / (1 + tau |K^|^2)
__global__ void blur_diag_kernel(const float2* __restrict__ khat, float tau, float* __restrict__ dgl, int n) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const float2 v = khat[e];
    dgl[e] = 1.f / (1.f + tau * (v.x * v.x + v.y * v.y));
  }
}

// ================================================================== phase retrieval (complex)
// rows forward: U[n][j][h][:] = FFT_row( D_j[h][:] * z[n][0][h][:] )
__global__ void __launch_bounds__(256) phase_rows_fwd_kernel(FftArgs f) {
  pdl_enter();
  extern __shared__ float2 sm2[];
  const int W = f.W, logW = f.logW;
  const int tpr = fft_tpr(W);
  const int rpb = 256 / tpr;
  float2* tw = sm2;
  float2* rows = sm2 + W / 2;
  load_twiddles(tw, f.tw_w, W);
  const int r = threadIdx.x / tpr, t = threadIdx.x % tpr;
  const int h = blockIdx.x * rpb + r;
  const int j = blockIdx.y, n = blockIdx.z;
  if (f.active && !f.active[n]) return;
  float2* d = rows + r * row_pitch(W);
  if (h < f.H) {
    const float* zr = f.z + (long long)n * f.H * W + (long long)h * W;
    const float2* Dr = f.pmask + ((long long)j * f.H + h) * W;
    for (int i = t; i < W; i += tpr) {
      const float zv = zr[i];
      const float2 dv = Dr[i];
      d[pd(bitrev(i, logW))] = make_float2(dv.x * zv, dv.y * zv);
    }
  }
  __syncthreads();
  fft_row(d, tw, W, logW, t, tpr, false);
  if (h < f.H) {
    float2* U = f.spec + (((long long)n * f.J + j) * f.H + h) * W;
    for (int i = t; i < W; i += tpr) U[i] = d[pd(i)];
  }
}

// columns: forward FFT -> u = col / sqrt(HW) (unitary) -> w = (|u|^2 - y_j) u -> inverse FFT
__global__ void __launch_bounds__(256) phase_cols_kernel(FftArgs f) {
  pdl_enter();
  extern __shared__ float2 sm2[];
  const int H = f.H, logH = f.logH, W = f.W;
  float2* tw = sm2;
  float2* cols = sm2 + H / 2;
  load_twiddles(tw, f.tw_h, H);
  const int tpc = 256 / FFT_CPB;
  const int cc = threadIdx.x / tpc, t = threadIdx.x % tpc;
  const int kx0 = blockIdx.x * FFT_CPB;
  const int j = blockIdx.y, n = blockIdx.z;
  if (f.active && !f.active[n]) return;
  float2* U = f.spec + ((long long)n * f.J + j) * H * W;
  const float* Y = f.y + ((long long)n * f.J + j) * H * W;
  for (int q = threadIdx.x; q < H * FFT_CPB; q += blockDim.x) {
    const int h = q / FFT_CPB, jj = q % FFT_CPB;
    cols[jj * col_pitch(H) + pd(bitrev(h, logH))] = U[(long long)h * W + kx0 + jj];
  }
  __syncthreads();
  float2* d = cols + cc * col_pitch(H);
  fft_row(d, tw, H, logH, t, tpc, false);
  const float s = rsqrtf((float)H * (float)W);
  const int kx = kx0 + cc;
  for (int ky = t; ky < H; ky += tpc) {
    const float2 v = d[pd(ky)];
    const float2 u = make_float2(v.x * s, v.y * s);
    const float m = u.x * u.x + u.y * u.y - Y[(long long)ky * W + kx];
    d[pd(ky)] = make_float2(m * u.x, m * u.y);
  }
  __syncthreads();
  bitrev_permute(d, H, logH, t, tpc);
  fft_row(d, tw, H, logH, t, tpc, true);
  for (int q = threadIdx.x; q < H * FFT_CPB; q += blockDim.x) {
    const int h = q / FFT_CPB, jj = q % FFT_CPB;
    U[(long long)h * W + kx0 + jj] = cols[jj * col_pitch(H) + pd(h)];
  }
}

// rows inverse: for each j, v = IFFT_row(U)/sqrt(HW); grad f += 2 Re(conj(D_j) v).
//   mode 0: store grad f into dst ; mode 1: x^{k+1} = z - tau (grad f + lam grad g) -> tail.
__global__ void __launch_bounds__(256) phase_rows_inv_kernel(FftArgs f, StepArgs a, float* __restrict__ dst, int mode) {
  pdl_enter();
  extern __shared__ float2 sm2[];
  const int W = f.W, logW = f.logW, H = f.H;
  const int tpr = fft_tpr(W);
  const int rpb = 256 / tpr;
  float2* tw = sm2;
  float2* rows = sm2 + W / 2;
  load_twiddles(tw, f.tw_w, W);
  const int r = threadIdx.x / tpr, t = threadIdx.x % tpr;
  const int h = blockIdx.x * rpb + r;
  const int n = blockIdx.y;
  if (f.active && !f.active[n]) return;
  float2* d = rows + r * row_pitch(W);
  constexpr int QMAX = 32;  // W / tpr <= 1024 / 32
  float gacc[QMAX];
#pragma unroll
  for (int q = 0; q < QMAX; ++q) gacc[q] = 0.f;
  const float s = rsqrtf((float)H * (float)W);
  for (int j = 0; j < f.J; ++j) {
    if (h < H) {
      const float2* U = f.spec + (((long long)n * f.J + j) * H + h) * W;
      for (int i = t; i < W; i += tpr) d[pd(bitrev(i, logW))] = U[i];
    }
    __syncthreads();
    fft_row(d, tw, W, logW, t, tpr, true);
    if (h < H) {
      const float2* Dr = f.pmask + ((long long)j * H + h) * W;
#pragma unroll
      for (int q = 0; q < QMAX; ++q) {
        const int i = t + q * tpr;
        if (i < W) {
          const float2 v = make_float2(d[pd(i)].x * s, d[pd(i)].y * s);
          gacc[q] += 2.f * cconjmul(Dr[i], v).x;
        }
      }
    }
    __syncthreads();
  }
  const long long base = (long long)n * H * W + (long long)h * W;
  if (mode == 0) {
    if (h < H) {
#pragma unroll
      for (int q = 0; q < QMAX; ++q)
        if (t + q * tpr < W) dst[base + t + q * tpr] = gacc[q];
    }
    return;
  }
  const int k = *a.kdev;
  const float* xk_base = (k & 1) ? a.X1 : a.X0;
  float* xn_base = (k & 1) ? a.X0 : a.X1;
  P3 acc{0.f, 0.f, 0.f};
  if (h < H) {
#pragma unroll
    for (int q = 0; q < QMAX; ++q) {
      const int i = t + q * tpr;
      if (i < W) {
        const long long e = base + i;
        // x^{k+1} = z - tau (grad f(z) + lam grad g(z))       (Alg. 1 l.8)
        step_tail(a.z[e] - a.tau * (gacc[q] + a.lam * a.gg[e]), e, a, xk_base, xn_base, acc);
      }
    }
  }
  reduce_store_p3(acc, a.partials + ((long long)n * a.parts + blockIdx.x) * 3);
}

// ================================================================== register FFTs (N = 256, 512)
// The shared-memory radix-2/4 passes above move each row through shared memory ~5 times per
// transform (~10 bytes of shared traffic per byte of HBM traffic: shared-memory bound at ~1 TB/s
// of HBM on B200). For the configs' sizes a transform of N = 16 T points is done by a TEAM of T
// threads (T = 16 for 256, 32 for 512) almost entirely in registers (four-step / Stockham):
//   thread t holds x[t + T k], k < 16 -> 16-point DFT in registers -> twiddle W_N^(t k') ->
//   one transpose through a padded per-team buffer -> a T-point DFT over the old thread index
//   (T = 16: one more 16-point DFT; T = 32: two 16-point DFTs over the even / odd samples joined
//   by one radix-2 step across a lane pair) -> thread holds X[n] for n = team_out(t, k).
// One shared-memory round trip per transform; loads and stores of x[t + T k] / X[team_out] are
// coalesced in 128-byte runs. Inverse transforms use conj(FFT(conj(x))). Twiddles: the
// fp64-derived table W_N^m, m < N/2 (tw_w / tw_h), with W_N^(m + N/2) = -W_N^m.
__device__ __forceinline__ float2 cfma_tw(float2 a, float c, float s) {  // a * (c + i s)
  return make_float2(a.x * c - a.y * s, a.x * s + a.y * c);
}
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }

// In-register 16-point DFT, natural order in and out (radix-2 decimation in frequency, the output
// permutation folded into register names at compile time).
__device__ __forceinline__ void dft16(float2 (&v)[16]) {
  // W_16^m, m < 8
  const float C[8] = {1.f, 0.92387953251128674f, 0.70710678118654752f, 0.38268343236508977f,
                      0.f, -0.38268343236508977f, -0.70710678118654752f, -0.92387953251128674f};
  const float S[8] = {0.f, -0.38268343236508977f, -0.70710678118654752f, -0.92387953251128674f,
                      -1.f, -0.92387953251128674f, -0.70710678118654752f, -0.38268343236508977f};
#pragma unroll
  for (int h = 8; h >= 1; h >>= 1) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if ((i & h) == 0) {
        const float2 a = v[i], b = v[i + h];
        v[i] = cadd(a, b);
        const int m = (i & (h - 1)) * (8 / h);
        v[i + h] = cfma_tw(csub(a, b), C[m], S[m]);
      }
    }
  }
  float2 o[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) o[k] = v[((k & 1) << 3) | ((k & 2) << 1) | ((k & 4) >> 1) | ((k & 8) >> 3)];
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = o[k];
}

__device__ __forceinline__ float2 tw_get(const float2* tw, int m, int N) {  // W_N^m for any m >= 0
  m &= N - 1;
  const float2 w = tw[m & (N / 2 - 1)];
  return m >= N / 2 ? make_float2(-w.x, -w.y) : w;
}

// Forward DFT of N = 16 T points held by a team of T threads: in v[k] = x[t + T k]; out v[k] =
// X[team_out<T>(t, k)]. buf: the team's (16 x (T + 1)) scratch; tw: W_N^m, m < N/2 (shared).
template <int T>
__device__ __forceinline__ int team_out(int t, int k) {
  if (T == 16) return t + 16 * k;
  return (t >> 1) + 16 * (k + 16 * (t & 1));
}
template <int T>
__device__ __forceinline__ void team_fft(float2 (&v)[16], int t, float2* buf, const float2* tw) {
  constexpr int N = 16 * T, P = T + 1;
  dft16(v);
#pragma unroll
  for (int k = 1; k < 16; ++k) v[k] = cmul(v[k], tw_get(tw, t * k, N));
#pragma unroll
  for (int k = 0; k < 16; ++k) buf[k * P + t] = v[k];
  __syncwarp();
  if (T == 16) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = buf[t * P + j];
    dft16(v);
  } else {
    const int kp = t >> 1, h = t & 1;
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = buf[kp * P + 2 * m + h];
    dft16(v);
    // X[k] = V0[k] + W_32^k V1[k], X[k + 16] = V0[k] - W_32^k V1[k]
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      float2 p;
      p.x = __shfl_xor_sync(0xffffffffu, v[k].x, 1);
      p.y = __shfl_xor_sync(0xffffffffu, v[k].y, 1);
      const float2 w = tw_get(tw, k * (N / 32), N);  // W_32^k
      v[k] = h ? csub(p, cmul(w, v[k])) : cadd(v[k], cmul(w, p));
    }
  }
  __syncwarp();  // the team buffer may be reused by the next transform
}

// Same transform with the team's transpose buffer laid over its OWN column of a column-pass tile
// (col[r * stride], r < 16 T: the column is in registers while the transform runs), skewed so
// both the column-wise writes and the row-wise reads are conflict-free: element (k, t) of the
// 16 x T buffer -> row T k + ((t + k) mod T). Frees the column passes' separate team buffers
// (a third of their shared memory), which doubles their occupancy.
template <int T>
__device__ __forceinline__ void team_fft_col(float2 (&v)[16], int t, float2* col, int stride, const float2* tw) {
  constexpr int N = 16 * T;
  auto at = [&](int k, int u) -> float2& { return col[(T * k + ((u + k) & (T - 1))) * stride]; };
  dft16(v);
#pragma unroll
  for (int k = 1; k < 16; ++k) v[k] = cmul(v[k], tw_get(tw, t * k, N));
#pragma unroll
  for (int k = 0; k < 16; ++k) at(k, t) = v[k];
  __syncwarp();
  if (T == 16) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = at(t, j);
    dft16(v);
  } else {
    const int kp = t >> 1, h = t & 1;
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = at(kp, 2 * m + h);
    dft16(v);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      float2 p;
      p.x = __shfl_xor_sync(0xffffffffu, v[k].x, 1);
      p.y = __shfl_xor_sync(0xffffffffu, v[k].y, 1);
      const float2 w = tw_get(tw, k * (N / 32), N);  // W_32^k
      v[k] = h ? csub(p, cmul(w, v[k])) : cadd(v[k], cmul(w, p));
    }
  }
  __syncwarp();  // the column is written by the caller next
}

// Row passes: RNT teams (rows) per block. Small blocks keep the grid many waves deep for the
// configs' small batches (C4: 16 images x 4 masks x 256 rows = 16384 row transforms).
constexpr int RNT = 4;

__device__ __forceinline__ void load_tw_all(float2* s_tw, const float2* g_tw, int N) {
  for (int k = threadIdx.x; k < N / 2; k += blockDim.x) s_tw[k] = g_tw[k];
}

// ---- blur / MRI rows (real planes): forward R2C (mode 0: src plane; 1: prox right-hand side)
template <int T>
__global__ void __launch_bounds__(RNT * T) rblur_rows_fwd_kernel(FftArgs f, const float* __restrict__ src, int mode) {
  pdl_enter();
  constexpr int W = 16 * T, P = T + 1;
  extern __shared__ float2 smr[];
  float2* tw = smr;                       // W/2
  float2 (*bufs)[16 * P] = reinterpret_cast<float2 (*)[16 * P]>(smr + W / 2);  // 16 teams
  load_tw_all(tw, f.tw_w, W);
  __syncthreads();
  const int team = threadIdx.x / T, t = threadIdx.x % T;
  const int h = blockIdx.x * RNT + team, c = blockIdx.y, n = blockIdx.z;
  if (f.active && !f.active[n]) return;  // uniform per block
  if (h >= f.H) return;                  // whole team
  const long long e0 = ((long long)n * f.C + c) * f.H * W + (long long)h * W;
  float2 v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const long long e = e0 + t + T * k;
    const float x = mode == 1 ? f.z[e] - f.tau * f.lam * f.gg[e] + f.tau * f.aty[e] : src[e];
    v[k] = make_float2(x, 0.f);
  }
  team_fft<T>(v, t, bufs[team], tw);
  const int Wh = W / 2 + 1;
  float2* S = f.spec + ((long long)n * f.C + c) * f.H * Wh + (long long)h * Wh;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int o = team_out<T>(t, k);
    if (o < Wh) S[o] = v[k];
  }
}

// ---- blur / MRI columns of the half spectrum: forward H-point FFT, op, inverse (as blur_cols)
template <int T>
__global__ void __launch_bounds__(256) rblur_cols_kernel(FftArgs f, int op) {
  pdl_enter();
  constexpr int H = 16 * T, CPB = 256 / T, CP = CPB + 1;  // CPB columns per block
  extern __shared__ float2 smc[];
  float2* tw = smc;                       // H/2
  float2* tile = smc + H / 2;             // [H][CP]; column j doubles as team j's FFT buffer
  float2* otile = tile + H * CP;          // [H][CPB] the op's diagonal (dgl as .x, or K^)
  load_tw_all(tw, f.tw_h, H);
  const int Wh = f.W / 2 + 1;
  const int kx0 = blockIdx.x * CPB, c = blockIdx.y, n = blockIdx.z;
  if (f.active && !f.active[n]) return;
  float2* S = f.spec + ((long long)n * f.C + c) * H * Wh;
  const bool diag = op == 0 || op == 1;
  // all of the strip's loads in flight at once (a load-then-store loop waited ~1 us per element)
  constexpr int NQ = H * CPB / 256;
  float2 lv[NQ], dv[NQ];
#pragma unroll
  for (int i = 0; i < NQ; ++i) {
    const int q = threadIdx.x + 256 * i, r = q / CPB, j = q % CPB;
    const bool in = kx0 + j < Wh;
    lv[i] = in ? S[(long long)r * Wh + kx0 + j] : make_float2(0.f, 0.f);
    dv[i] = make_float2(0.f, 0.f);
    if (diag && in)
      dv[i] = op == 0 ? make_float2(__ldg(f.dgl + (long long)r * Wh + kx0 + j), 0.f)
                      : __ldg(f.khat + (long long)r * Wh + kx0 + j);
  }
#pragma unroll
  for (int i = 0; i < NQ; ++i) {
    const int q = threadIdx.x + 256 * i, r = q / CPB, j = q % CPB;
    tile[r * CP + j] = lv[i];
    if (diag) otile[q] = dv[i];
  }
  __syncthreads();
  const int team = threadIdx.x / T, t = threadIdx.x % T;
  const int kx = kx0 + team;
  float2* col = tile + team;
  float2 v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = tile[(t + T * k) * CP + team];
  const bool fwd = op != 3, inv = op != 2;
  if (fwd) team_fft_col<T>(v, t, col, CP, tw);
  if (fwd && inv) {  // pointwise op at ky = team_out, then back to the x[t + T k] distribution
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int ky = team_out<T>(t, k);
      float2 w = v[k];
      if (kx < Wh) {
        const float2 o = otile[ky * CPB + team];
        if (op == 0) {
          w.x *= o.x; w.y *= o.x;
        } else {
          w = cconjmul(o, w);
        }
      }
      tile[ky * CP + team] = w;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = tile[(t + T * k) * CP + team];
  }
  if (inv) {
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = cconj(v[k]);
    team_fft_col<T>(v, t, col, CP, tw);
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = cconj(v[k]);
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 16; ++k) tile[team_out<T>(t, k) * CP + team] = v[k];
  __syncthreads();
  for (int q = threadIdx.x; q < H * CPB; q += blockDim.x) {
    const int r = q / CPB, j = q % CPB;
    if (kx0 + j < Wh) S[(long long)r * Wh + kx0 + j] = tile[r * CP + j];
  }
}

// ---- blur / MRI rows, inverse C2R (mode 0: store into dst; 1: x^{k+1} -> update + partials)
template <int T>
__global__ void __launch_bounds__(RNT * T) rblur_rows_inv_kernel(FftArgs f, StepArgs a, float* __restrict__ dst, int mode) {
  pdl_enter();
  constexpr int W = 16 * T, P = T + 1;
  extern __shared__ float2 smr[];
  float2* tw = smr;                       // W/2
  float2 (*bufs)[16 * P] = reinterpret_cast<float2 (*)[16 * P]>(smr + W / 2);  // 16 teams
  load_tw_all(tw, f.tw_w, W);
  __syncthreads();
  const int team = threadIdx.x / T, t = threadIdx.x % T;
  const int c = blockIdx.y, n = blockIdx.z, H = f.H;
  const bool valid = blockIdx.x * RNT + team < H;
  const int h = valid ? blockIdx.x * RNT + team : H - 1;  // rows past H (H < RNT) redo row H-1, unused
  if (f.active && !f.active[n]) return;
  const int Wh = W / 2 + 1;
  const float2* S = f.spec + ((long long)n * f.C + c) * H * Wh + (long long)h * Wh;
  float2 v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {  // Hermitian row: X[W - i] = conj(X[i]); loaded conjugated (inverse)
    const int i = t + T * k;
    const float2 x = i < Wh ? S[i] : cconj(S[W - i]);
    v[k] = cconj(x);
  }
  team_fft<T>(v, t, bufs[team], tw);
  const float scale = 1.f / ((float)H * (float)W);
  const long long plane = ((long long)n * f.C + c) * H * W + (long long)h * W;
  if (mode == 0) {
    if (valid)
#pragma unroll
      for (int k = 0; k < 16; ++k) dst[plane + team_out<T>(t, k)] = v[k].x * scale;  // Re(conj(.)) = Re(.)
    return;
  }
  const int kk = *a.kdev;
  const float* xk_base = (kk & 1) ? a.X1 : a.X0;
  float* xn_base = (kk & 1) ? a.X0 : a.X1;
  P3 acc{0.f, 0.f, 0.f};
  if (valid)
#pragma unroll
    for (int k = 0; k < 16; ++k) step_tail(v[k].x * scale, plane + team_out<T>(t, k), a, xk_base, xn_base, acc);
  const int part = c * gridDim.x + blockIdx.x;
  reduce_store_p3(acc, a.partials + ((long long)n * a.parts + part) * 3);
}

// ---- phase retrieval rows forward: U[n][j][h][:] = FFT_row(D_j[h][:] z[n][h][:])
template <int T>
__global__ void __launch_bounds__(RNT * T) rphase_rows_fwd_kernel(FftArgs f) {
  pdl_enter();
  constexpr int W = 16 * T, P = T + 1;
  extern __shared__ float2 smr[];
  float2* tw = smr;                       // W/2
  float2 (*bufs)[16 * P] = reinterpret_cast<float2 (*)[16 * P]>(smr + W / 2);  // 16 teams
  load_tw_all(tw, f.tw_w, W);
  __syncthreads();
  const int team = threadIdx.x / T, t = threadIdx.x % T;
  const int h = blockIdx.x * RNT + team, j = blockIdx.y, n = blockIdx.z;
  if (f.active && !f.active[n]) return;
  if (h >= f.H) return;  // whole team
  const float* zr = f.z + (long long)n * f.H * W + (long long)h * W;
  const float2* Dr = f.pmask + ((long long)j * f.H + h) * W;
  float2 v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int i = t + T * k;
    const float zv = zr[i];
    const float2 dv = __ldg(Dr + i);
    v[k] = make_float2(dv.x * zv, dv.y * zv);
  }
  team_fft<T>(v, t, bufs[team], tw);
  float2* U = f.spec + (((long long)n * f.J + j) * f.H + h) * W;
#pragma unroll
  for (int k = 0; k < 16; ++k) U[team_out<T>(t, k)] = v[k];
}

// ---- phase columns: forward FFT -> u = col / sqrt(HW) -> w = (|u|^2 - y_j) u -> inverse FFT
template <int T>
__global__ void __launch_bounds__(256) rphase_cols_kernel(FftArgs f) {
  pdl_enter();
  constexpr int H = 16 * T, CPB = 256 / T, CP = CPB + 1;
  extern __shared__ float2 smc[];
  float2* tw = smc;
  float2* tile = smc + H / 2;  // [H][CP]; column j doubles as team j's FFT buffer
  float* ytile = reinterpret_cast<float*>(tile + H * CP);  // [H][CPB]
  load_tw_all(tw, f.tw_h, H);
  const int W = f.W;
  const int kx0 = blockIdx.x * CPB, j = blockIdx.y, n = blockIdx.z;
  if (f.active && !f.active[n]) return;
  float2* U = f.spec + ((long long)n * f.J + j) * H * W;
  const float* Y = f.y + ((long long)n * f.J + j) * H * W;
  constexpr int NQ = H * CPB / 256;  // all of the strip's loads in flight at once
  float2 lv[NQ];
  float yv[NQ];
#pragma unroll
  for (int i = 0; i < NQ; ++i) {
    const int q = threadIdx.x + 256 * i, r = q / CPB, jj = q % CPB;
    lv[i] = U[(long long)r * W + kx0 + jj];
    yv[i] = __ldg(Y + (long long)r * W + kx0 + jj);
  }
#pragma unroll
  for (int i = 0; i < NQ; ++i) {
    const int q = threadIdx.x + 256 * i, r = q / CPB, jj = q % CPB;
    tile[r * CP + jj] = lv[i];
    ytile[q] = yv[i];
  }
  __syncthreads();
  const int team = threadIdx.x / T, t = threadIdx.x % T;
  float2* col = tile + team;
  float2 v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = tile[(t + T * k) * CP + team];
  team_fft_col<T>(v, t, col, CP, tw);
  const float sc = rsqrtf((float)H * (float)W);
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int ky = team_out<T>(t, k);
    const float2 u = make_float2(v[k].x * sc, v[k].y * sc);
    const float m = u.x * u.x + u.y * u.y - ytile[ky * CPB + team];
    tile[ky * CP + team] = make_float2(m * u.x, m * u.y);
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = cconj(tile[(t + T * k) * CP + team]);
  team_fft_col<T>(v, t, col, CP, tw);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 16; ++k) tile[team_out<T>(t, k) * CP + team] = cconj(v[k]);
  __syncthreads();
  for (int q = threadIdx.x; q < H * CPB; q += blockDim.x) {
    const int r = q / CPB, jj = q % CPB;
    U[(long long)r * W + kx0 + jj] = tile[r * CP + jj];
  }
}

// ---- phase rows inverse: v_j = IFFT_row(U_j) / sqrt(HW); grad f = sum_j 2 Re(conj(D_j) v_j). One
// team per (row, mask): a block is RB = NTI / J rows x J masks (NTI = 4 for J <= 4, else 16; J a
// power of two <= 16); the J contributions of a pixel are summed in a fixed order through shared
// memory before the update.
template <int T, int NTI>
__global__ void __launch_bounds__(NTI * T) rphase_rows_inv_kernel(FftArgs f, StepArgs a, float* __restrict__ dst, int mode) {
  pdl_enter();
  constexpr int W = 16 * T, P = T + 1;
  extern __shared__ float2 smr[];
  float2* tw = smr;
  float2 (*bufs)[16 * P] = reinterpret_cast<float2 (*)[16 * P]>(smr + W / 2);
  float* gsum = reinterpret_cast<float*>(smr + W / 2 + NTI * 16 * P);  // [NTI teams][W]
  load_tw_all(tw, f.tw_w, W);
  __syncthreads();
  const int J = f.J, RB = NTI / J;
  const int team = threadIdx.x / T, t = threadIdx.x % T;
  const int rl = team / J, j = team % J;
  const int n = blockIdx.y, H = f.H;
  const int h = blockIdx.x * RB + rl < H ? blockIdx.x * RB + rl : H - 1;  // rows past H: redo the last, unused
  if (f.active && !f.active[n]) return;
  const float sc = rsqrtf((float)H * (float)W);
  {
    const float2* U = f.spec + (((long long)n * J + j) * H + h) * W;
    float2 v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = cconj(U[t + T * k]);
    team_fft<T>(v, t, bufs[team], tw);
    const float2* Dr = f.pmask + ((long long)j * H + h) * W;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int o = team_out<T>(t, k);
      const float2 w = make_float2(v[k].x * sc, -v[k].y * sc);  // conj back
      gsum[team * W + o] = 2.f * cconjmul(__ldg(Dr + o), w).x;
    }
  }
  __syncthreads();
  // per pixel of the block's RB rows: fixed-order sum over the masks, then store / update
  const long long base0 = (long long)n * H * W + (long long)blockIdx.x * RB * W;
  const int kk = mode == 1 ? *a.kdev : 0;  // the component call (mode 0) passes no solver state
  const float* xk_base = (kk & 1) ? a.X1 : a.X0;
  float* xn_base = (kk & 1) ? a.X0 : a.X1;
  P3 acc{0.f, 0.f, 0.f};
  const int rows = H - (int)blockIdx.x * RB < RB ? H - (int)blockIdx.x * RB : RB;
  for (int q = threadIdx.x; q < rows * W; q += blockDim.x) {
    const int r = q / W, i = q % W;
    float g = 0.f;
    for (int jj = 0; jj < J; ++jj) g += gsum[(r * J + jj) * W + i];
    const long long e = base0 + (long long)r * W + i;
    if (mode == 0) dst[e] = g;
    // x^{k+1} = z - tau (grad f(z) + lam grad g(z))       (Alg. 1 l.8)
    else step_tail(a.z[e] - a.tau * (g + a.lam * a.gg[e]), e, a, xk_base, xn_base, acc);
  }
  if (mode == 1) reduce_store_p3(acc, a.partials + ((long long)n * a.parts + blockIdx.x) * 3);
}

static bool reg_n(int N) { return N == 256 || N == 512; }
template <int T, int NT = RNT>
static size_t rrow_smem() { return sizeof(float2) * ((size_t)8 * T + (size_t)NT * 16 * (T + 1)); }
template <int T, int NTI>
static size_t rpinv_smem() { return rrow_smem<T, NTI>() + sizeof(float) * (size_t)NTI * 16 * T; }
static bool phase_j_ok(int J) { return J >= 1 && J <= 16 && (16 % J) == 0; }
template <int T>
static size_t rcol_smem() {
  constexpr int CPB = 256 / T;  // twiddles, tile (its columns are the team buffers), op / observation tile
  return sizeof(float2) * ((size_t)8 * T + (size_t)16 * T * (CPB + 1) + (size_t)16 * T * CPB);
}

// ------------------------------------------------------------------ launchers
static int ilog2(int v) { int l = 0; while ((1 << l) < v) ++l; return l; }

static size_t row_smem(int W) {
  const int tpr = fft_tpr(W);
  const int rpb = 256 / tpr;
  return sizeof(float2) * (W / 2 + (size_t)rpb * row_pitch(W));
}
static size_t col_smem(int H) { return sizeof(float2) * (H / 2 + (size_t)FFT_CPB * col_pitch(H)); }
static int rows_per_block(int W) { return 256 / fft_tpr(W); }            // shared-memory row passes
static int rows_per_block_any(int W) { return reg_n(W) ? RNT : rows_per_block(W); }  // the pass launched

int fft_parts_per_image(int C, int H, int W) { return C * ((H + rows_per_block_any(W) - 1) / rows_per_block_any(W)); }
// the register row pass of phase retrieval covers 16 / J rows per block (J <= 16 masks)
static int phase_nti(int J) { return J <= 4 ? 4 : 16; }
int phase_parts_per_image(int H, int W, int J) {
  return (reg_n(W) && phase_j_ok(J)) ? (H * J + phase_nti(J) - 1) / phase_nti(J)
                                     : (H + rows_per_block(W) - 1) / rows_per_block(W);
}

bool fft_size_ok(int H, int W) {
  auto pow2 = [](int v) { return v >= 4 && v <= 1024 && (v & (v - 1)) == 0; };
  return pow2(H) && pow2(W);
}

void fft_fill_args(FftArgs& f) { f.logH = ilog2(f.H); f.logW = ilog2(f.W); }

void launch_blur_rows_fwd(const FftArgs& f, const float* src, int mode, int N, cudaStream_t s) {
  dim3 grid((f.H + rows_per_block_any(f.W) - 1) / rows_per_block_any(f.W), f.C, N);
  if (f.W == 256) { launch_k(rblur_rows_fwd_kernel<16>, grid, RNT * 16, rrow_smem<16>(), s, f, src, mode); return; }
  if (f.W == 512) { launch_k(rblur_rows_fwd_kernel<32>, grid, RNT * 32, rrow_smem<32>(), s, f, src, mode); return; }
  launch_k(blur_rows_fwd_kernel, grid, 256, row_smem(f.W), s, f, src, mode);
}
void launch_blur_cols(const FftArgs& f, int op, int N, cudaStream_t s) {
  if (reg_n(f.H)) {
    const int cpb = f.H == 256 ? 16 : 8;
    dim3 g((f.W / 2 + 1 + cpb - 1) / cpb, f.C, N);
    if (f.H == 256) launch_k(rblur_cols_kernel<16>, g, 256, rcol_smem<16>(), s, f, op);
    else launch_k(rblur_cols_kernel<32>, g, 256, rcol_smem<32>(), s, f, op);
    return;
  }
  dim3 grid((f.W / 2 + 1 + FFT_CPB - 1) / FFT_CPB, f.C, N);
  launch_k(blur_cols_kernel, grid, 256, col_smem(f.H), s, f, op);
}
void launch_blur_rows_inv(const FftArgs& f, const StepArgs& a, float* dst, int mode, int N, cudaStream_t s) {
  dim3 grid((f.H + rows_per_block_any(f.W) - 1) / rows_per_block_any(f.W), f.C, N);
  if (f.W == 256) { launch_k(rblur_rows_inv_kernel<16>, grid, RNT * 16, rrow_smem<16>(), s, f, a, dst, mode); return; }
  if (f.W == 512) { launch_k(rblur_rows_inv_kernel<32>, grid, RNT * 32, rrow_smem<32>(), s, f, a, dst, mode); return; }
  launch_k(blur_rows_inv_kernel, grid, 256, row_smem(f.W), s, f, a, dst, mode);
}
void launch_embed_kernel(const float* k, int ks, float* plane, int H, int W, cudaStream_t s) {
  cudaMemsetAsync(plane, 0, sizeof(float) * H * W, s);
  embed_kernel_kernel<<<(ks * ks + 255) / 256, 256, 0, s>>>(k, ks, plane, H, W);
}
void launch_mri_fill(const float* y, const uint8_t* kmask, float2* spec, int N, int H, int W, float scale,
                     cudaStream_t s) {
  const int n = H * (W / 2 + 1);
  mri_fill_kernel<<<dim3((n + 255) / 256, N), 256, 0, s>>>(y, kmask, spec, H, W, scale);
}
void launch_mri_masks(const uint8_t* kmask, float* mhalf, float* dgl, float tau, int H, int W, cudaStream_t s) {
  const int n = H * (W / 2 + 1);
  mri_masks_kernel<<<(n + 255) / 256, 256, 0, s>>>(kmask, mhalf, dgl, tau, H, W);
}
void launch_blur_diag(const float2* khat, float tau, float* dgl, int n, cudaStream_t s) {
  blur_diag_kernel<<<(n + 255) / 256, 256, 0, s>>>(khat, tau, dgl, n);
}
void launch_phase_rows_fwd(const FftArgs& f, int N, cudaStream_t s) {
  dim3 grid((f.H + rows_per_block_any(f.W) - 1) / rows_per_block_any(f.W), f.J, N);
  if (f.W == 256) { launch_k(rphase_rows_fwd_kernel<16>, grid, RNT * 16, rrow_smem<16>(), s, f); return; }
  if (f.W == 512) { launch_k(rphase_rows_fwd_kernel<32>, grid, RNT * 32, rrow_smem<32>(), s, f); return; }
  launch_k(phase_rows_fwd_kernel, grid, 256, row_smem(f.W), s, f);
}
void launch_phase_cols(const FftArgs& f, int N, cudaStream_t s) {
  if (reg_n(f.H) && f.W % 16 == 0) {
    const int cpb = f.H == 256 ? 16 : 8;
    dim3 g(f.W / cpb, f.J, N);
    if (f.H == 256) launch_k(rphase_cols_kernel<16>, g, 256, rcol_smem<16>(), s, f);
    else launch_k(rphase_cols_kernel<32>, g, 256, rcol_smem<32>(), s, f);
    return;
  }
  dim3 grid(f.W / FFT_CPB, f.J, N);
  launch_k(phase_cols_kernel, grid, 256, col_smem(f.H), s, f);
}
void launch_phase_rows_inv(const FftArgs& f, const StepArgs& a, float* dst, int mode, int N, cudaStream_t s) {
  if (reg_n(f.W) && phase_j_ok(f.J)) {
    const int nti = phase_nti(f.J);
    dim3 g((f.H * f.J + nti - 1) / nti, N);
    if (nti == 4) {
      if (f.W == 256) launch_k(rphase_rows_inv_kernel<16, 4>, g, 64, rpinv_smem<16, 4>(), s, f, a, dst, mode);
      else launch_k(rphase_rows_inv_kernel<32, 4>, g, 128, rpinv_smem<32, 4>(), s, f, a, dst, mode);
    } else {
      if (f.W == 256) launch_k(rphase_rows_inv_kernel<16, 16>, g, 256, rpinv_smem<16, 16>(), s, f, a, dst, mode);
      else launch_k(rphase_rows_inv_kernel<32, 16>, g, 512, rpinv_smem<32, 16>(), s, f, a, dst, mode);
    }
    return;
  }
  dim3 grid((f.H + rows_per_block(f.W) - 1) / rows_per_block(f.W), N);
  launch_k(phase_rows_inv_kernel, grid, 256, row_smem(f.W), s, f, a, dst, mode);
}

void init_attrs_fft() {
  set_max_dyn_smem(rblur_rows_fwd_kernel<16>);
  set_max_dyn_smem(rblur_rows_fwd_kernel<32>);
  set_max_dyn_smem(rblur_rows_inv_kernel<16>);
  set_max_dyn_smem(rblur_rows_inv_kernel<32>);
  set_max_dyn_smem(rphase_rows_fwd_kernel<16>);
  set_max_dyn_smem(rphase_rows_fwd_kernel<32>);
  set_max_dyn_smem(rphase_rows_inv_kernel<16, 4>);
  set_max_dyn_smem(rphase_rows_inv_kernel<32, 4>);
  set_max_dyn_smem(rphase_rows_inv_kernel<16, 16>);
  set_max_dyn_smem(rphase_rows_inv_kernel<32, 16>);
  set_max_dyn_smem(rblur_cols_kernel<16>);
  set_max_dyn_smem(rblur_cols_kernel<32>);
  set_max_dyn_smem(rphase_cols_kernel<16>);
  set_max_dyn_smem(rphase_cols_kernel<32>);
  set_max_dyn_smem(blur_rows_fwd_kernel);
  set_max_dyn_smem(blur_cols_kernel);
  set_max_dyn_smem(blur_rows_inv_kernel);
  set_max_dyn_smem(phase_rows_fwd_kernel);
  set_max_dyn_smem(phase_cols_kernel);
  set_max_dyn_smem(phase_rows_inv_kernel);
}

}  // namespace ideq
