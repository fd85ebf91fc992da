// Microbenchmark: tcgen05.mma (kind::f16, bf16 -> f32, cta_group::1, M = 128, SS operands)
// issue rate versus N, with operands resident in shared memory (no loads). Measures cycles
// per MMA for N in {32, 64, 96, 128, 192, 256} with the A start aligned to the 1024-B swizzle
// atom or shifted by one 128-B row (the row-shifted halo windows of conv_tc.cu).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_bench tools/umma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

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

__global__ void __launch_bounds__(128, 1) umma_rate(int n, int iters, int shift_rows, int kc64, int mode, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tmem_holder;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_holder)),
                 "r"(256u) : "memory");
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
  if (mode == 1 && warp == 0) {
    // whole warp runs the loop (warp-uniform descriptor math in uniform registers); one elected
    // lane issues; descriptors advance by adding (bytes >> 4) to the 64-bit value
    const uint32_t layout = kc64 ? 2u : 4u, sbo = kc64 ? 1024u : 512u, rowb = kc64 ? 128u : 64u;
    const uint32_t a0 = base + (uint32_t)shift_rows * rowb;
    const uint32_t b0 = base + 40 * 1024;
    const uint64_t ad0 = make_sdesc(a0, sbo, layout), bd0 = make_sdesc(b0, sbo, layout);
    const uint32_t idesc = make_idesc_bf16(n);
    const int ksteps = kc64 ? 4 : 2;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (k < ksteps) {
          asm volatile(
              "{\n\t.reg .pred p, e;\n\t"
              "elect.sync _|e, 0xffffffff;\n\t"
              "setp.ne.b32 p, %4, 0;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
              "l"(ad0 + 2ull * k), "l"(bd0 + 2ull * k), "r"(idesc), "r"(1)
              : "memory");
        }
      }
    }
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                   : "memory");
      asm volatile(
          "{\n\t.reg .pred p;\nW1:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W1;\n}\n" ::"r"(
              smem_u32(&bar))
          : "memory");
      long long t1 = clock64();
      out[blockIdx.x] = t1 - t0;
    }
    __syncwarp();
  }
  if (mode == 0 && threadIdx.x == 0) {
    const uint32_t layout = kc64 ? 2u : 4u, sbo = kc64 ? 1024u : 512u, rowb = kc64 ? 128u : 64u;
    const uint32_t a0 = base + (uint32_t)shift_rows * rowb;  // A: 128 rows (+ shift) x KC
    const uint32_t b0 = base + 40 * 1024;                    // B: n rows x KC
    const uint32_t idesc = make_idesc_bf16(n);
    const int ksteps = kc64 ? 4 : 2;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int k = 0; k < ksteps; ++k) {
        const uint64_t ad = make_sdesc(a0 + 32u * k, sbo, layout);
        const uint64_t bd = make_sdesc(b0 + 32u * k, sbo, layout);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"(1)
            : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}\n" ::"r"(
            smem_u32(&bar))
        : "memory");
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256u) : "memory");
}

int main() {
  long long* d;
  cudaMalloc(&d, 1024 * sizeof(long long));
  cudaFuncSetAttribute(umma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 2048;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mode = 0; mode <= 1; ++mode)
  for (int kc64 = 0; kc64 <= 1; ++kc64)
    for (int shift = 0; shift <= (mode ? 0 : 1); ++shift)
      for (int n : {32, 64, 96, 128, 192, 256}) {
        for (int g : {sms}) {
          umma_rate<<<g, 128, 100 * 1024>>>(n, iters, shift, kc64, mode, d);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
          long long h[1024];
          cudaMemcpy(h, d, g * sizeof(long long), cudaMemcpyDeviceToHost);
          long long mx = 0;
          for (int i = 0; i < g; ++i) mx = h[i] > mx ? h[i] : mx;
          const double mmas = (double)iters * (kc64 ? 4 : 2);
          printf("mode=%d KC=%d shift=%d N=%3d grid=%3d : %.1f clk/MMA (floor %.1f) -> %.0f%% of floor rate\n", mode, kc64 ? 64 : 32,
                 shift, n, g, mx / mmas, 128.0 * n / 256.0, 100.0 * (128.0 * n / 256.0) / (mx / mmas));
        }
      }
  return 0;
}
