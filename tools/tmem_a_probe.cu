// Probe: tcgen05.mma with the A operand in TENSOR MEMORY (kind::f16, "TS" form), fed by
// tcgen05.cp 128x256b from a SW64 K-major shared-memory tile at row-shifted (pixel-shifted)
// starts -- the building block of a level-0 convolution whose activation operand is read once
// from shared memory per input row instead of once per MMA.
//   1. correctness: D_dw = X[dw .. dw+127] . W^T for dw = 0, 1, 2 (cp from shifted windows);
//      in-order hazard: mma(D3, A0); cp(new -> A0); mma(D4, A0) must give old / new products
//   2. throughput: clk per TS MMA at N = 32 / 64, clk per tcgen05.cp 128x256b
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_a_probe tools/tmem_a_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)(1u) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(layout & 7u) << 61;
  return d;
}
__device__ __forceinline__ uint32_t make_idesc_bf16(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void cp128x256(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void mma_ts_e(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_ss_e(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void cp_e(uint32_t taddr, uint64_t sdesc) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n\t}\n"
               ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void commit_wait(uint32_t bar, uint32_t& ph) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
  asm volatile(
      "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n}\n" ::"r"(bar),
      "r"(ph)
      : "memory");
  ph ^= 1u;
}
// SW64 K-major tile: 64-byte rows (32 bf16), 16-byte chunk j of row r at j ^ ((r >> 1) & 3)
__device__ __forceinline__ uint32_t sw64(uint32_t base, int r, int j) {
  return base + (uint32_t)r * 64u + (uint32_t)((j ^ ((r >> 1) & 3)) << 4);
}

// X: [136][32] bf16 (global, row-major), X2: a second version for the hazard test, W: [32][32]
__global__ void __launch_bounds__(128, 1) probe(const __nv_bfloat16* X, const __nv_bfloat16* X2,
                                                const __nv_bfloat16* W, float* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tmem_holder;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  unsigned char* g = smem + (base - smem_u32(smem));
  const uint32_t sX = base, sX2 = base + 16 * 1024, sW = base + 32 * 1024;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 136 * 4; i += 128) {
    const int r = i >> 2, j = i & 3;
    *reinterpret_cast<uint4*>(g + (sw64(sX, r, j) - base)) = *reinterpret_cast<const uint4*>(X + r * 32 + j * 8);
    *reinterpret_cast<uint4*>(g + (sw64(sX2, r, j) - base)) = *reinterpret_cast<const uint4*>(X2 + r * 32 + j * 8);
  }
  for (int i = threadIdx.x; i < 32 * 4; i += 128) {
    const int r = i >> 2, j = i & 3;
    *reinterpret_cast<uint4*>(g + (sw64(sW, r, j) - base)) = *reinterpret_cast<const uint4*>(W + r * 32 + j * 8);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_holder)),
                 "r"(512u) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_holder;
  const uint32_t idesc = make_idesc_bf16(32);
  uint32_t ph = 0;
  if (threadIdx.x == 0) {
    const uint64_t wd = make_sdesc(sW, 512u, 4u);
    // A slots at columns 256 + dw*16 + k*8; D_dw at columns dw*32
    for (int dw = 0; dw < 3; ++dw)
      for (int k = 0; k < 2; ++k) cp128x256(tmem + 256 + dw * 16 + k * 8, make_sdesc(sX + dw * 64 + k * 32, 512u, 4u));
    for (int dw = 0; dw < 3; ++dw)
      for (int k = 0; k < 2; ++k) mma_ts(tmem + dw * 32, tmem + 256 + dw * 16 + k * 8, wd + 2ull * k, idesc, k);
    // SS reference for dw = 1 (the known-good shifted-descriptor MMA) into D at columns 96..127
    for (int k = 0; k < 2; ++k) mma_ss(tmem + 96, make_sdesc(sX + 64 + k * 32, 512u, 4u), wd + 2ull * k, idesc, k);
    // hazard: mma(D4 @128, A slot dw=0); cp X2 -> the same slot; mma(D5 @160, same slot)
    for (int k = 0; k < 2; ++k) mma_ts(tmem + 128, tmem + 256 + k * 8, wd + 2ull * k, idesc, k);
    for (int k = 0; k < 2; ++k) cp128x256(tmem + 256 + k * 8, make_sdesc(sX2 + k * 32, 512u, 4u));
    for (int k = 0; k < 2; ++k) mma_ts(tmem + 160, tmem + 256 + k * 8, wd + 2ull * k, idesc, k);
    commit_wait(smem_u32(&bar), ph);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // D blocks 0..5 (32 columns each): out[blk][m][n]
  for (int blk = 0; blk < 6; ++blk) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(tmem + ((uint32_t)(warp * 32) << 16) + blk * 32));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int m = warp * 32 + lane;
    for (int n = 0; n < 32; ++n) out[(blk * 128 + m) * 32 + n] = __uint_as_float(r[n]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
}

// throughput: mode 0 = TS MMA (A in TMEM), mode 1 = SS MMA (A in smem), mode 2 = cp 128x256b,
// mode 3 = conv row pattern: per "row" 6 cp + 18 TS MMAs
__global__ void __launch_bounds__(128, 1) rate(int n, int iters, int mode, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tmem_holder;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_holder)),
                 "r"(512u) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_holder;
  if (warp == 0) {
    const uint32_t idesc = make_idesc_bf16(n);
    const uint64_t ad = make_sdesc(base, 512u, 4u), bd = make_sdesc(base + 32 * 1024, 512u, 4u);
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (mode == 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k) mma_ts_e(tmem, tmem + 256 + k * 8, bd + 2ull * (k & 1), idesc, 1);
      } else if (mode == 1) {
#pragma unroll
        for (int k = 0; k < 8; ++k) mma_ss_e(tmem, ad + 2ull * (k & 1), bd + 2ull * (k & 1), idesc, 1);
      } else if (mode == 2) {
#pragma unroll
        for (int k = 0; k < 8; ++k) cp_e(tmem + 256 + k * 8, ad + 2ull * (k & 1));
      } else {
        const uint32_t slot = (uint32_t)(it & 3) * 48u;
#pragma unroll
        for (int k = 0; k < 6; ++k) cp_e(tmem + 256 + ((slot + k * 8) % 192), ad + 4ull * k);
#pragma unroll
        for (int k = 0; k < 18; ++k) mma_ts_e(tmem + (it & 3) * 32, tmem + 256 + ((k * 8) % 192), bd + 2ull * (k & 1), idesc, 1);
      }
    }
    if (threadIdx.x == 0) {
      commit_wait(smem_u32(&bar), ph);
      out[blockIdx.x] = clock64() - t0;
    }
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
}

static float bf(float x) { return __bfloat162float(__float2bfloat16(x)); }

int main() {
  std::vector<__nv_bfloat16> X(136 * 32), X2(136 * 32), W(32 * 32);
  std::vector<float> xf(136 * 32), x2f(136 * 32), wf(32 * 32);
  srand(1);
  for (int i = 0; i < 136 * 32; ++i) {
    xf[i] = bf((float)(rand() % 9 - 4) * 0.5f);
    x2f[i] = bf((float)(rand() % 9 - 4) * 0.25f);
    X[i] = __float2bfloat16(xf[i]);
    X2[i] = __float2bfloat16(x2f[i]);
  }
  for (int i = 0; i < 32 * 32; ++i) { wf[i] = bf((float)(rand() % 7 - 3)); W[i] = __float2bfloat16(wf[i]); }
  __nv_bfloat16 *dX, *dX2, *dW;
  float* dout;
  cudaMalloc(&dX, X.size() * 2); cudaMalloc(&dX2, X2.size() * 2); cudaMalloc(&dW, W.size() * 2);
  cudaMalloc(&dout, 6 * 128 * 32 * 4);
  cudaMemcpy(dX, X.data(), X.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dX2, X2.data(), X2.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dW, W.data(), W.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe<<<1, 128, 64 * 1024>>>(dX, dX2, dW, dout);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("probe error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> o(6 * 128 * 32);
  cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
  auto ref = [&](const std::vector<float>& x, int dw, int m, int n) {
    double s = 0;
    for (int c = 0; c < 32; ++c) s += (double)x[(m + dw) * 32 + c] * wf[n * 32 + c];
    return s;
  };
  const char* names[6] = {"TS dw=0", "TS dw=1", "TS dw=2", "SS dw=1", "hazard old", "hazard new"};
  for (int blk = 0; blk < 6; ++blk) {
    double maxerr = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 32; ++n) {
        const int dw = blk < 3 ? blk : (blk == 3 ? 1 : 0);
        const double r = ref(blk == 5 ? x2f : xf, dw, m, n);
        maxerr = fmax(maxerr, fabs(r - o[(blk * 128 + m) * 32 + n]));
      }
    printf("%-11s max|err| = %g %s\n", names[blk], maxerr, maxerr == 0 ? "OK" : "MISMATCH");
  }
  long long* d;
  cudaMalloc(&d, 1024 * sizeof(long long));
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 1024;
  const char* mn[4] = {"TS mma", "SS mma", "cp 128x256b", "row: 6cp+18TS"};
  for (int mode = 0; mode < 4; ++mode)
    for (int n : {32, 64}) {
      rate<<<sms, 128, 70 * 1024>>>(n, iters, mode, d);
      e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("rate error %s\n", cudaGetErrorString(e)); return 1; }
      long long h[1024];
      cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
      const double per = mode == 3 ? 24.0 : 8.0;
      printf("%-14s N=%d : %.1f clk per op (%s)\n", mn[mode], n, (double)mx / iters / per,
             mode == 3 ? "per cp/mma op; x24 = per 128-px row" : "");
    }
  return 0;
}
