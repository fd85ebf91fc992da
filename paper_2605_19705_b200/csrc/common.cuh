// Shared device/host definitions of the i-DEQ CUDA library (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "this library targets sm_100a (B200) only"
#endif

namespace ideq {

// ---------------------------------------------------------------- element types
template <typename T> struct ElemOps;
template <> struct ElemOps<float> {
  static __device__ __forceinline__ float ld(const float* p) { return *p; }
  static __device__ __forceinline__ void st(float* p, float v) { *p = v; }
};
template <> struct ElemOps<__nv_bfloat16> {
  static __device__ __forceinline__ float ld(const __nv_bfloat16* p) { return __bfloat162float(*p); }
  static __device__ __forceinline__ void st(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
};

// ---------------------------------------------------------------- activations
// softplus (beta = 1, no threshold; reading Q20) and its derivative from the SAVED
// ACTIVATION a = sp(p): sigmoid(p) = 1 - exp(-a), so the VJP never needs p itself.
__device__ __forceinline__ float softplus_f(float t) {
  return fmaxf(t, 0.f) + log1pf(__expf(-fabsf(t)));
}
__device__ __forceinline__ float dsoftplus_from_act(float a) { return -expm1f(-a); }

// ---------------------------------------------------------------- epilogue modes
enum Epi : int {
  EPI_STORE = 0,     // out = acc
  EPI_SOFTPLUS = 1,  // out = sp(acc)                       (RB conv A forward; saved)
  EPI_RESADD = 2,    // out = acc + aux                     (RB conv B fwd / conv A^T, skip adds)
  EPI_SIGMUL = 3,    // out = acc * sp'(.) from aux = saved activation   (conv B^T)
  EPI_IMG = 4,       // tcgen05 only: columns [0, C) -> fp32 NCHW image planes, + alpha * aux image
};

// ---------------------------------------------------------------- division by a runtime constant
// q = n / d for 0 <= n < 2^31 with one IMAD.HI + add + shift (no I2F/MUFU.RCP/F2I on the XU
// pipe, which the per-tile index math of the persistent conv kernels otherwise saturates).
struct FastDiv {
  uint32_t d, m, s;
  __host__ void init(uint32_t div) {
    d = div < 1 ? 1 : div;
    s = 0;
    while ((1u << s) < d) ++s;
    m = (uint32_t)((((1ull << 32) * ((1ull << s) - d)) / d) + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, m) + n) >> s; }
};

// ---------------------------------------------------------------- implicit-GEMM geometry
// The input tensor is viewed as a 5-D NHWC array (C', W', P, H', N): element
// (c, w, p, h, n) sits at ((((n*H' + h)*P + p)*W' + w)*C' + c).
//   conv3x3 / 1x1 : C'=C, W'=W, P=1, H'=H
//   2x2 stride-2 patch on a fine grid : C'=2C (pixel pair along W), W'=W/2, P=2 (row parity), H'=H/2
// Output pixels form an (OH, OW) grid tiled by R rows x Wt columns (R*Wt <= 128).
// K-block kb = tap * nchunk + chunk reads channels [chunk*KC, +KC) at input pixel
// (h + dh[tap], w + dw[tap]) of parity plane p[tap]; out of range => 0 (conv padding).
// GEMM column col (< ncols) of output pixel (n, oh, ow) is written at
//   ((n*OHo + oh*osh + col / CB)*OWo + ow*osw)*OCp + col % CB
// which covers the plain NHWC store (osh=osw=1, CB=OCp=ncols) and the 2x2 pixel
// scatter of the transposed / adjoint strided convs (osh=osw=2, CB=2*OCp).
struct ConvGeom {
  int N;
  int inC, inW, inP, inH;
  int OH, OW, R, Wt, tiles_h, tiles_w;
  int ncols, KC, nchunk, ntaps;
  int dh[9], dw[9], dp[9];
  int OHo, OWo, osh, osw, OCp, CB;
  int epi;
};

__host__ __device__ __forceinline__ long long out_offset(const ConvGeom& g, int n, int oh, int ow, int col) {
  return ((long long)(n * g.OHo + oh * g.osh + col / g.CB) * g.OWo + (long long)ow * g.osw) * g.OCp + col % g.CB;
}

__device__ __forceinline__ float apply_epi(int epi, float acc, float aux) {
  switch (epi) {
    case EPI_SOFTPLUS: return softplus_f(acc);
    case EPI_RESADD: return acc + aux;
    case EPI_SIGMUL: return acc * dsoftplus_from_act(aux);
    default: return acc;
  }
}

// Programmatic dependent launch for the per-iteration kernels: launched with the programmatic
// stream-serialization attribute, each waits (griddepcontrol.wait) for its predecessor grid to
// complete and flush before touching any global data, then lets its own successor be scheduled,
// so the launch latency of the next kernel overlaps this one. Opt-in: IDEQ_PDL_SMALL=1 (step.cu).
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Allow a kernel the largest dynamic shared memory the device grants on top of its
// static shared memory (the opt-in limit is per block, static + dynamic).
template <typename K>
inline void set_max_dyn_smem(K kernel) {
  cudaFuncAttributes a;
  if (cudaFuncGetAttributes(&a, kernel) != cudaSuccess) { cudaGetLastError(); return; }
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)a.sharedSizeBytes);
  cudaGetLastError();
}

}  // namespace ideq
