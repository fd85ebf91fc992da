// Kernels of the JFB training gradient at x_hat, fp32 FFMA path.
//
// dL/dtheta = -tau lam d/dtheta <v, grad g_theta(z)>, and with the identity skip
// <v, grad g> = <U'(z)[v], U(z)>: the network runs forward on the primal z and the tangent v,
// then one reverse pass over both streams collects the weight gradients (oracle/jfb.py is the
// fp64 reference). This file holds the pieces the runtime (ideq_api.cu) strings together:
//   - weight gradient of any implicit-GEMM layer, in the layer's own [kb][ncols][KC] operand
//     layout (the runtime maps it back to the blob order),
//   - weight gradients of the image <-> feature head / tail convolutions,
//   - softplus forward / tangent / reverse (with the sp'' cross term) element kernels,
//   - the JFB residual (T, r, v) and fixed-order dot products.
#include "common.cuh"
#include "kernels.h"

namespace ideq {

// dB[kb][col][k] += sum_{n, oh, ow} in(n, oh + dh[tap], ow + dw[tap], dp[tap], chunk*KC + k)
//                                    * gout[out_offset(n, oh, ow, col)]
// i.e. the gradient of <gout, layer(in)> w.r.t. the layer's GEMM operand B: per tap a
// [ncols x ktap] = G^T A contraction over the N*OH*OW output pixels. Tiled FFMA GEMM: a CTA owns a
// TM x TN (cols x channels) tile of one tap and a contiguous pixel range (blockIdx.y); each step
// stages P = 32 pixels of G (gout columns) and A (shifted input channels, float4 loads) in shared
// memory, every thread accumulates a 4 x 4 register block. Partials per pixel range are summed in
// range order by wgrad_sum_kernel (fixed order: deterministic).
template <int TM, int TN>
__global__ void __launch_bounds__(TM * TN / 16) wgrad_tile_kernel(ConvGeom g, const float* __restrict__ in,
                                                                  const float* __restrict__ gout,
                                                                  float* __restrict__ part, long long per, int ktap) {
  constexpr int P = 32, NT = TM * TN / 16, TX = TN / 4;
  __shared__ __align__(16) float sG[P][TM];
  __shared__ __align__(16) float sA[P][TN];
  __shared__ long long sGo[P], sAo[P];
  const int ncb = g.ncols / TM, nkb = ktap / TN;
  int bid = blockIdx.x;
  const int cb = bid % ncb;
  bid /= ncb;
  const int kb2 = bid % nkb, tap = bid / nkb;
  const int col0 = cb * TM, c0 = kb2 * TN;
  const long long npix = (long long)g.N * g.OH * g.OW;
  const long long q0 = blockIdx.y * per, q1 = q0 + per < npix ? q0 + per : npix;
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (long long qb = q0; qb < q1; qb += P) {
    for (int p = tid; p < P; p += NT) {
      const long long q = qb + p;
      long long go = -1, ao = -1;
      if (q < q1) {
        const int ow = (int)(q % g.OW);
        const long long r = q / g.OW;
        const int oh = (int)(r % g.OH), n = (int)(r / g.OH);
        go = out_offset(g, n, oh, ow, 0);
        const int h = oh + g.dh[tap], w = ow + g.dw[tap];
        if (h >= 0 && h < g.inH && w >= 0 && w < g.inW)
          ao = ((((long long)n * g.inH + h) * g.inP + g.dp[tap]) * g.inW + w) * g.inC;
      }
      sGo[p] = go;
      sAo[p] = ao;
    }
    __syncthreads();
    for (int e = tid; e < P * TN / 4; e += NT) {
      const int p = e / (TN / 4), c4 = e % (TN / 4);
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (sAo[p] >= 0) v = __ldg(reinterpret_cast<const float4*>(in + sAo[p] + c0 + c4 * 4));
      *reinterpret_cast<float4*>(&sA[p][c4 * 4]) = v;
    }
    for (int e = tid; e < P * TM; e += NT) {
      const int p = e / TM, cc = e % TM, col = col0 + cc;
      float v = 0.f;
      if (sGo[p] >= 0) v = __ldg(gout + sGo[p] + (long long)(col / g.CB) * g.OWo * g.OCp + col % g.CB);
      sG[p][cc] = v;
    }
    __syncthreads();
#pragma unroll 8
    for (int p = 0; p < P; ++p) {
      const float4 gv = *reinterpret_cast<const float4*>(&sG[p][ty * 4]);
      const float4 av = *reinterpret_cast<const float4*>(&sA[p][tx * 4]);
      const float gg[4] = {gv.x, gv.y, gv.z, gv.w}, aa[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(gg[i], aa[j], acc[i][j]);
    }
    __syncthreads();
  }
  const long long total = (long long)g.ntaps * g.nchunk * g.ncols * g.KC;
  float* dst = part + blockIdx.y * total;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int col = col0 + ty * 4 + i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + tx * 4 + j;
      dst[((long long)(tap * g.nchunk + c / g.KC) * g.ncols + col) * g.KC + c % g.KC] = acc[i][j];
    }
  }
}
__global__ void wgrad_sum_kernel(const float* __restrict__ part, int S, long long total, float* __restrict__ dB) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < S; ++s) acc += part[s * total + i];
    dB[i] += acc;
  }
}

static int tile_dim(int n) { return n % 64 == 0 ? 64 : n % 32 == 0 ? 32 : 16; }
// pixel ranges: ~2048 threads per SM of (tile, range) CTAs, each range >= 128 pixels
static int wgrad_splits(const ConvGeom& g, long long* per_out) {
  const int ktap = g.nchunk * g.KC, TM = tile_dim(g.ncols), TN = tile_dim(ktap);
  const long long blocks = (long long)g.ntaps * (g.ncols / TM) * (ktap / TN), nt = TM * TN / 16;
  const long long npix = (long long)g.N * g.OH * g.OW;
  long long S = (148LL * 2048 + blocks * nt - 1) / (blocks * nt);
  const long long smax = (npix + 127) / 128;
  if (S > smax) S = smax;
  if (S > 1024) S = 1024;
  if (S < 1) S = 1;
  const long long per = (npix + S - 1) / S;
  if (per_out) *per_out = per;
  return (int)((npix + per - 1) / per);
}
size_t wgrad_workspace(const ConvGeom& g) {
  const long long total = (long long)g.ntaps * g.nchunk * g.ncols * g.KC;
  return (size_t)wgrad_splits(g, nullptr) * total;
}
template <int TM, int TN>
static void wgrad_tile(const ConvGeom& g, const float* in, const float* gout, float* ws, long long per, int S,
                       cudaStream_t s) {
  const int ktap = g.nchunk * g.KC;
  const unsigned blocks = (unsigned)(g.ntaps * (g.ncols / TM) * (ktap / TN));
  wgrad_tile_kernel<TM, TN><<<dim3(blocks, S), TM * TN / 16, 0, s>>>(g, in, gout, ws, per, ktap);
}
template <int TM>
static void wgrad_tile_n(int TN, const ConvGeom& g, const float* in, const float* gout, float* ws, long long per,
                         int S, cudaStream_t s) {
  if (TN == 64) wgrad_tile<TM, 64>(g, in, gout, ws, per, S, s);
  else if (TN == 32) wgrad_tile<TM, 32>(g, in, gout, ws, per, S, s);
  else wgrad_tile<TM, 16>(g, in, gout, ws, per, S, s);
}
void launch_wgrad_geom(const ConvGeom& g, const float* in, const float* gout, float* dB, float* ws, cudaStream_t s) {
  const long long total = (long long)g.ntaps * g.nchunk * g.ncols * g.KC;
  long long per = 0;
  const int S = wgrad_splits(g, &per);
  const int TM = tile_dim(g.ncols), TN = tile_dim(g.nchunk * g.KC);
  if (TM == 64) wgrad_tile_n<64>(TN, g, in, gout, ws, per, S, s);
  else if (TM == 32) wgrad_tile_n<32>(TN, g, in, gout, ws, per, S, s);
  else wgrad_tile_n<16>(TN, g, in, gout, ws, per, S, s);
  long long gb = (total + 255) / 256;
  wgrad_sum_kernel<<<(unsigned)(gb > 148 * 8 ? 148 * 8 : gb), 256, 0, s>>>(ws, S, total, dB);
}

// head (image -> features): f[n][h][w][co] = sum W[co][ci][a][b] img[n][ci][h+a-1][w+b-1]
// dW[co][ci][a][b] += sum_{n,h,w} gf[n][h][w][co] * img[n][ci][h+a-1][w+b-1]
// tail (features -> image): img[n][c][h][w] = sum W[c][ci][a][b] f[n][h+a-1][w+b-1][ci]
// dW[c][ci][a][b] += sum gimg[n][c][h][w] * f[n][h+a-1][w+b-1][ci]
// Same two-pass split as above, over ranges of the N*H image rows.
template <bool TAIL>
__global__ void headtail_wgrad_kernel(const float* __restrict__ x, const float* __restrict__ g,
                                      float* __restrict__ part, int N, int C, int H, int W, int wf, int per) {
  const int total = wf * C * 9;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int o = idx / ((TAIL ? wf : C) * 9), i = (idx / 9) % (TAIL ? wf : C), a = (idx % 9) / 3, b = idx % 3;
  const int r0 = blockIdx.y * per, r1 = min(r0 + per, N * H);
  float acc = 0.f;
  for (int r = r0; r < r1; ++r) {
    const int n = r / H, h = r % H, hh = h + a - 1;
    if (hh < 0 || hh >= H) continue;
    for (int w = 0; w < W; ++w) {
      const int ww = w + b - 1;
      if (ww < 0 || ww >= W) continue;
      if (!TAIL)  // o = co (feature), i = ci (image channel)
        acc = fmaf(g[(((long long)n * H + h) * W + w) * wf + o], x[(((long long)n * C + i) * H + hh) * W + ww], acc);
      else        // o = c (image channel), i = ci (feature)
        acc = fmaf(g[(((long long)n * C + o) * H + h) * W + w], x[(((long long)n * H + hh) * W + ww) * wf + i], acc);
    }
  }
  part[(long long)blockIdx.y * total + idx] = acc;
}

static int headtail_splits(int N, int H) { return N * H < 2048 ? N * H : 2048; }
size_t headtail_wgrad_workspace(int N, int C, int H, int wf) { return (size_t)headtail_splits(N, H) * wf * C * 9; }

template <bool TAIL>
static void launch_headtail_wgrad(const float* x, const float* g, float* dW, float* ws, int N, int C, int H, int W,
                                  int wf, cudaStream_t s) {
  const int total = wf * C * 9;
  const int S0 = headtail_splits(N, H), per = (N * H + S0 - 1) / S0, S = (N * H + per - 1) / per;
  headtail_wgrad_kernel<TAIL><<<dim3((total + 127) / 128, S), 128, 0, s>>>(x, g, ws, N, C, H, W, wf, per);
  wgrad_sum_kernel<<<(total + 255) / 256, 256, 0, s>>>(ws, S, total, dW);
}
void launch_head_wgrad(const float* img, const float* gf, float* dW, float* ws, int N, int C, int H, int W, int wf,
                       cudaStream_t s) {
  launch_headtail_wgrad<false>(img, gf, dW, ws, N, C, H, W, wf, s);
}
void launch_tail_wgrad(const float* f, const float* gimg, float* dW, float* ws, int N, int C, int H, int W, int wf,
                       cudaStream_t s) {
  launch_headtail_wgrad<true>(f, gimg, dW, ws, N, C, H, W, wf, s);
}

// ---- softplus pieces (s = sp'(p) = 1 - exp(-a) from a = sp(p), reading R1; sp'' = s (1 - s))
__global__ void sp_forward_kernel(const float* __restrict__ p, float* __restrict__ a, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    a[i] = softplus_f(p[i]);
}
// a_dot = sp'(p) p_dot
__global__ void sp_tangent_kernel(const float* __restrict__ a, const float* __restrict__ pd, float* __restrict__ ad,
                                  long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    ad[i] = dsoftplus_from_act(a[i]) * pd[i];
}
// p_dot_bar = s a_dot_bar ; p_bar = s a_bar + s (1 - s) p_dot a_dot_bar
__global__ void sp_reverse_kernel(const float* __restrict__ a, const float* __restrict__ pd,
                                  const float* __restrict__ ab, const float* __restrict__ adb, float* __restrict__ pb,
                                  float* __restrict__ pdb, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float s = dsoftplus_from_act(a[i]);
    pdb[i] = s * adb[i];
    pb[i] = s * ab[i] + s * (1.f - s) * pd[i] * adb[i];
  }
}
static unsigned ew_grid(long long n) {
  long long g = (n + 255) / 256;
  return (unsigned)(g > 148 * 8 ? 148 * 8 : (g < 1 ? 1 : g));
}
void launch_sp_forward(const float* p, float* a, long long n, cudaStream_t s) {
  sp_forward_kernel<<<ew_grid(n), 256, 0, s>>>(p, a, n);
}
void launch_sp_tangent(const float* a, const float* pd, float* ad, long long n, cudaStream_t s) {
  sp_tangent_kernel<<<ew_grid(n), 256, 0, s>>>(a, pd, ad, n);
}
void launch_sp_reverse(const float* a, const float* pd, const float* ab, const float* adb, float* pb, float* pdb,
                       long long n, cudaStream_t s) {
  sp_reverse_kernel<<<ew_grid(n), 256, 0, s>>>(a, pd, ab, adb, pb, pdb, n);
}
__global__ void scale_kernel(float* __restrict__ x, float s, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    x[i] *= s;
}
void launch_scale(float* x, float s, long long n, cudaStream_t st) { scale_kernel<<<ew_grid(n), 256, 0, st>>>(x, s, n); }

// ---- JFB residual at z = x_hat: per element
//   gradient step: T = z - tau (gf + lam gg), r = T - x*, v = r,
//                  dlam term -tau gg r, dtau term -(gf + lam gg) r
//   inpainting prox: vin = z - tau lam gg, T = (tau m y + vin) / (tau m + 1), r = T - x*,
//                  v = r / (1 + tau m), dlam term -tau gg v,
//                  dtau term r [(m y - lam gg) / (1 + tau m) - (tau m y + vin) m / (1 + tau m)^2]
// writes v and three per-element terms (0.5 r^2, dlam, dtau) for the fixed-order reductions.
__global__ void jfb_residual_kernel(const float* __restrict__ z, const float* __restrict__ xs,
                                    const float* __restrict__ gg, const float* __restrict__ gf,
                                    const float* __restrict__ y, const uint8_t* __restrict__ mask, int prox,
                                    float lam, float tau, long long n, long long HW, long long CHW,
                                    float* __restrict__ v, float* __restrict__ terms) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float r, vv, tl, tt;
    if (!prox) {
      const float T = z[i] - tau * (gf[i] + lam * gg[i]);
      r = T - xs[i];
      vv = r;
      tl = -tau * gg[i] * r;
      tt = -(gf[i] + lam * gg[i]) * r;
    } else {
      const float m = (float)mask[(i / CHW) * HW + (i % HW)];
      const float vin = z[i] - tau * lam * gg[i];
      const float den = 1.f + tau * m;
      const float T = (tau * m * y[i] + vin) / den;
      r = T - xs[i];
      vv = r / den;
      tl = -tau * gg[i] * vv;
      tt = r * ((m * y[i] - lam * gg[i]) / den - (tau * m * y[i] + vin) * m / (den * den));
    }
    v[i] = vv;
    terms[i] = 0.5f * r * r;
    terms[n + i] = tl;
    terms[2 * n + i] = tt;
  }
}
void launch_jfb_residual(const float* z, const float* xs, const float* gg, const float* gf, const float* y,
                         const uint8_t* mask, int prox, float lam, float tau, long long n, long long HW, long long CHW,
                         float* v, float* terms, cudaStream_t s) {
  jfb_residual_kernel<<<ew_grid(n), 256, 0, s>>>(z, xs, gg, gf, y, mask, prox, lam, tau, n, HW, CHW, v, terms);
}

// Fixed-order sums of `k` consecutive length-n vectors: block partials (grid-stride, fp64), then
// one block combines them in index order.
__global__ void dot_partials_kernel(const float* __restrict__ x, long long n, double* __restrict__ part) {
  __shared__ double red[256];
  const int j = blockIdx.y;
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    acc += (double)x[j * n + i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[j * gridDim.x + blockIdx.x] = red[0];
}
__global__ void dot_final_kernel(const double* __restrict__ part, int nb, int k, double* __restrict__ out) {
  const int j = threadIdx.x;
  if (j >= k) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += part[j * nb + b];
  out[j] = s;
}
void launch_sums(const float* x, long long n, int k, double* part, double* out, cudaStream_t s) {
  const int nb = 256;
  dot_partials_kernel<<<dim3(nb, k), 256, 0, s>>>(x, n, part);
  dot_final_kernel<<<1, 32, 0, s>>>(part, nb, k, out);
}

}  // namespace ideq
