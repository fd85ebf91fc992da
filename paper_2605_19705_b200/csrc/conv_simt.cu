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
// Tile: 128 output pixels (the same R x Wt pixel tile the tcgen05 path uses) x 64 GEMM
// columns; 256 threads, 8 pixels x 4 columns each; K staged 16 channels at a time.
constexpr int SM_BM = 128, SM_BN = 64, SM_BK = 16;

template <typename T>
__global__ void __launch_bounds__(256) conv_simt_kernel(ConvGeom g, const T* __restrict__ in,
                                                        const T* __restrict__ wB, T* __restrict__ out,
                                                        const T* __restrict__ aux) {
  __shared__ __align__(16) float As[SM_BK][SM_BM + 4];
  __shared__ __align__(16) float Bs[SM_BK][SM_BN + 4];
  const int tid = threadIdx.x;
  const int mt = blockIdx.x;
  const int n0 = blockIdx.y * SM_BN;
  const int per_img = g.tiles_h * g.tiles_w;
  const int img = mt / per_img;
  const int th = (mt % per_img) / g.tiles_w, tw = mt % g.tiles_w;
  const int oh0 = th * g.R, ow0 = tw * g.Wt;
  const int tile_px = g.R * g.Wt;

  // A-load role: pixel lpx, 8 channels starting at lhalf*8
  const int lpx = tid >> 1, lhalf = tid & 1;
  const int loh = oh0 + lpx / g.Wt, low = ow0 + lpx % g.Wt;
  const bool lvalid = lpx < tile_px && loh < g.OH && low < g.OW;
  // B-load role: column bcol, 4 k-values starting at bk
  const int bcol = tid >> 2, bk = (tid & 3) * 4;
  const bool bvalid = (n0 + bcol) < g.ncols;

  // compute role
  const int ty = tid >> 4, tx = tid & 15;
  float acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  const int nkb = g.ntaps * g.nchunk;
  for (int kb = 0; kb < nkb; ++kb) {
    const int tap = kb / g.nchunk, chunk = kb % g.nchunk;
    const int ih = loh + g.dh[tap], iw = low + g.dw[tap];
    const bool inb = lvalid && ih >= 0 && ih < g.inH && iw >= 0 && iw < g.inW;
    const T* src = in + ((((long long)img * g.inH + ih) * g.inP + g.dp[tap]) * g.inW + iw) * g.inC + chunk * g.KC;
    const T* wsrc = wB + ((long long)kb * g.ncols + n0 + bcol) * g.KC;
    for (int kk = 0; kk < g.KC; kk += SM_BK) {
#pragma unroll
      for (int j = 0; j < 8; ++j) As[lhalf * 8 + j][lpx] = inb ? ElemOps<T>::ld(src + kk + lhalf * 8 + j) : 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) Bs[bk + j][bcol] = bvalid ? ElemOps<T>::ld(wsrc + kk + bk + j) : 0.f;
      __syncthreads();
#pragma unroll
      for (int k = 0; k < SM_BK; ++k) {
        const float4 a0 = *reinterpret_cast<const float4*>(&As[k][ty * 8]);
        const float4 a1 = *reinterpret_cast<const float4*>(&As[k][ty * 8 + 4]);
        const float4 b = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
        const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      __syncthreads();
    }
  }
  // epilogue
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int px = ty * 8 + i;
    const int oh = oh0 + px / g.Wt, ow = ow0 + px % g.Wt;
    if (px >= tile_px || oh >= g.OH || ow >= g.OW) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = n0 + tx * 4 + j;
      if (col >= g.ncols) continue;
      const long long o = out_offset(g, img, oh, ow, col);
      const float av = (g.epi == EPI_RESADD || g.epi == EPI_SIGMUL) ? ElemOps<T>::ld(aux + o) : 0.f;
      ElemOps<T>::st(out + o, apply_epi(g.epi, acc[i][j], av));
    }
  }
}

template <typename T>
void launch_conv_simt(const ConvGeom& g, const T* in, const T* wB, T* out, const T* aux, cudaStream_t s) {
  dim3 grid(g.N * g.tiles_h * g.tiles_w, (g.ncols + SM_BN - 1) / SM_BN);
  conv_simt_kernel<T><<<grid, 256, 0, s>>>(g, in, wB, out, aux);
}

// ------------------------------------------------------------------ head-side: image -> features
// out[n,h,w,co] = epi( sum_{ci,a,b} w_t[co][ci][a][b] in[n,ci,h+a-1,w+b-1] ), zero padding.
template <typename T, int WO>
__global__ void __launch_bounds__(256) img2feat_kernel(const float* __restrict__ in, const float* __restrict__ w_t,
                                                       T* __restrict__ out, const T* __restrict__ aux, int epi,
                                                       int N, int C, int H, int W) {
  __shared__ float wsm[WO * 3 * 9];
  for (int t = threadIdx.x; t < WO * C * 9; t += blockDim.x) {
    const int co = t / (C * 9), r = t % (C * 9);
    wsm[r * WO + co] = w_t[t];  // [ci*9 + a*3 + b][co]
  }
  __syncthreads();
  const long long pix = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long HW = (long long)H * W;
  if (pix >= (long long)N * HW) return;
  const int n = (int)(pix / HW);
  const int h = (int)((pix % HW) / W), w = (int)(pix % W);
  float acc[WO];
#pragma unroll
  for (int co = 0; co < WO; ++co) acc[co] = 0.f;
  for (int ci = 0; ci < C; ++ci) {
    const float* plane = in + ((long long)n * C + ci) * HW;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const int hh = h + a - 1, ww = w + b - 1;
        const float v = (hh >= 0 && hh < H && ww >= 0 && ww < W) ? plane[(long long)hh * W + ww] : 0.f;
        const float* wr = wsm + (ci * 9 + a * 3 + b) * WO;
#pragma unroll
        for (int co = 0; co < WO; ++co) acc[co] = fmaf(wr[co], v, acc[co]);
      }
    }
  }
  T* o = out + pix * WO;
  const T* x = aux ? aux + pix * WO : nullptr;
#pragma unroll
  for (int co = 0; co < WO; ++co) {
    const float av = x ? ElemOps<T>::ld(x + co) : 0.f;
    ElemOps<T>::st(o + co, apply_epi(epi, acc[co], av));
  }
}

template <typename T>
void launch_img2feat(const float* in, const float* w_t, T* out, const T* aux, int epi, int N, int C, int H, int W,
                     int wout, cudaStream_t s) {
  const long long P = (long long)N * H * W;
  const unsigned blocks = (unsigned)((P + 255) / 256);
  switch (wout) {
    case 16: img2feat_kernel<T, 16><<<blocks, 256, 0, s>>>(in, w_t, out, aux, epi, N, C, H, W); break;
    case 32: img2feat_kernel<T, 32><<<blocks, 256, 0, s>>>(in, w_t, out, aux, epi, N, C, H, W); break;
    case 64: img2feat_kernel<T, 64><<<blocks, 256, 0, s>>>(in, w_t, out, aux, epi, N, C, H, W); break;
    default: break;  // rejected by the runtime at create
  }
}

// ------------------------------------------------------------------ tail-side: features -> image
// out[n,c,h,w] = sum_{ci,a,b} w_t[c][ci][a][b] in[n,h+a-1,w+b-1,ci] + alpha * aux[n,c,h,w]
// 16x16 output pixels per block; input tile 18x18xWI staged in shared memory.
template <typename T, int WI>
__global__ void __launch_bounds__(256) feat2img_kernel(const T* __restrict__ in, const float* __restrict__ w_t,
                                                       float* __restrict__ out, const float* __restrict__ aux,
                                                       float alpha, int N, int C, int H, int W) {
  extern __shared__ __align__(16) unsigned char smraw[];
  float* wsm = reinterpret_cast<float*>(smraw);                  // [C][9][WI]
  constexpr int PS = WI + (sizeof(T) == 4 ? 1 : 2);              // padded pixel stride (bank spread)
  T* tile = reinterpret_cast<T*>(smraw + sizeof(float) * 3 * 9 * WI);  // [18][18][PS]
  const int n = blockIdx.z;
  const int h0 = blockIdx.y * 16, w0 = blockIdx.x * 16;
  for (int t = threadIdx.x; t < C * WI * 9; t += blockDim.x) {
    const int c = t / (WI * 9), r = t % (WI * 9);
    const int ci = r / 9, ab = r % 9;
    wsm[(c * 9 + ab) * WI + ci] = w_t[t];
  }
  const T zero = T(0.f);
  for (int t = threadIdx.x; t < 18 * 18 * WI; t += blockDim.x) {
    const int ci = t % WI, q = t / WI;
    const int u = q / 18, v = q % 18;
    const int hh = h0 + u - 1, ww = w0 + v - 1;
    tile[q * PS + ci] = (hh >= 0 && hh < H && ww >= 0 && ww < W) ? in[(((long long)n * H + hh) * W + ww) * WI + ci] : zero;
  }
  __syncthreads();
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  const int h = h0 + ty, w = w0 + tx;
  float acc[3] = {0.f, 0.f, 0.f};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const T* tp = tile + ((ty + a) * 18 + (tx + b)) * PS;
      for (int ci = 0; ci < WI; ++ci) {
        const float v = ElemOps<T>::ld(tp + ci);
        for (int c = 0; c < C; ++c) acc[c] = fmaf(wsm[(c * 9 + a * 3 + b) * WI + ci], v, acc[c]);
      }
    }
  }
  if (h >= H || w >= W) return;
  const long long HW = (long long)H * W;
  for (int c = 0; c < C; ++c) {
    const long long o = ((long long)n * C + c) * HW + (long long)h * W + w;
    out[o] = acc[c] + (aux ? alpha * aux[o] : 0.f);
  }
}

template <typename T>
void launch_feat2img(const T* in, const float* w_t, float* out, const float* aux, float alpha, int N, int C, int H,
                     int W, int win, cudaStream_t s) {
  dim3 grid((W + 15) / 16, (H + 15) / 16, N);
  const size_t sm = sizeof(float) * 3 * 9 * win + sizeof(T) * 18 * 18 * (win + 2);
  switch (win) {
#define F2I(WI)                                                                                                \
  case WI:                                                                                                     \
    feat2img_kernel<T, WI><<<grid, 256, sm, s>>>(in, w_t, out, aux, alpha, N, C, H, W);                        \
    break;
    F2I(16) F2I(32) F2I(64)
#undef F2I
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
