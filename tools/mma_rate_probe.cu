// Probe: tcgen05.mma kind::f16 throughput (M = 128, K = 16 per instruction): clk per MMA by N,
// operand swizzle, A start alignment, accumulator / A-tile rotation and operand data (zero or not).
// One CTA per SM, one warp issues (elect.sync) NIT x 8 MMAs; clock64 around issue + commit wait.
// Inter-warp interference modes (inter 1..5): TMEM loads / stores and shared-memory traffic from
// three other warps while the MMAs run.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_rate_probe tools/mma_rate_probe.cu
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
__device__ __forceinline__ void mma_e(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t}\n" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc)
      : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

constexpr int NIT = 512;
// layout 4 = SW64 (64-byte rows), 2 = SW128 (128-byte rows); rotD / rotA: cycle 4 accumulators /
// 4 A tiles per group of 8 MMAs; shift: A start + 1 row; data: fill value of the operands
__global__ void probe(int layout, int n, int shift, int rotD, int rotA, uint32_t data, int mode, int inter, int sboA,
                      const uint4* __restrict__ gsrc, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
  unsigned char* g = sm + (base - smem_u32(sm));
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t bar2;
  __shared__ uint32_t tm;
  __shared__ volatile int stop_flag;
  const uint32_t rowb = layout == 4 ? 64u : 128u, sbo = 8u * rowb;
  for (uint32_t o = threadIdx.x * 4; o < 96u * 1024u; o += blockDim.x * 4) {  // operands
    uint32_t v = data;
    if (data == 1u) {  // pseudo-random bf16 pairs in [-1, 1)
      uint32_t h = (o + 0x9e3779b9u * (blockIdx.x + 1)) * 2654435761u;
      h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
      v = (0x3f80u | ((h & 0x7fu) << 0) | ((h >> 7 & 1u) << 15)) | ((0x3f00u | (h >> 8 & 0x7fu) | ((h >> 15 & 1u) << 15)) << 16);
    }
    *(uint32_t*)(g + o) = v;
  }
  if (threadIdx.x == 0) {
    stop_flag = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tm)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tm;
  if (threadIdx.x < 32) {
    const uint32_t idesc = make_idesc_bf16(n);
    const uint64_t bd = make_sdesc(base + 64u * 1024u, sbo, (uint32_t)layout);
    uint64_t ad[4];
    // sboA != 0: A's 8-row core groups sboA bytes apart (the halo tiles' (Wt + 2) x row bytes)
    const uint32_t sa = sboA ? (uint32_t)sboA : sbo;
    for (int t = 0; t < 4; ++t)
      ad[t] = make_sdesc(base + (uint32_t)t * (sboA ? 2048u : 128u * rowb) + (uint32_t)shift * rowb, sa, (uint32_t)layout);
    const uint32_t dstep = n <= 128 ? 128u : 256u;
    const long long t0 = clock64();
    for (int it = 0; it < NIT; ++it) {
      const uint32_t d = tmem + (rotD ? (uint32_t)(it & (n <= 128 ? 3 : 1)) * dstep : 0u);
      const uint64_t a = rotA ? ad[it & 3] : ad[0];
      if (mode == 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k) mma_e(d, a + 2ull * (k & 1), bd + 2ull * (k & 1), idesc);
      } else if (mode == 1) {  // N cycles 96, 64, 32
#pragma unroll
        for (int k = 0; k < 8; ++k) mma_e(d, a + 2ull * (k & 1), bd + 2ull * (k & 1), make_idesc_bf16(96 - 32 * (k % 3)));
      } else if (mode == 2) {  // A start cycles -1, 0, +1 rows (4 = 64 B in 16-byte units)
#pragma unroll
        for (int k = 0; k < 8; ++k) mma_e(d, a + 4ull * (k % 3) + 2ull * (k & 1), bd + 2ull * (k & 1), idesc);
      } else if (mode == 4 || mode == 5) {  // kernel-like: 6 N=96 MMAs then a commit (mode 5: + a fence)
#pragma unroll
        for (int k = 0; k < 6; ++k) mma_e(d, a + 4ull * (k >> 1) + 2ull * (k & 1), bd + 2ull * (k & 1), idesc);
        if (threadIdx.x == 0) commit(smem_u32(&bar2));
        if (mode == 5) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      } else if (mode >= 10) {  // D column offset (mode - 10) * 32 within a 128-column group
#pragma unroll
        for (int k = 0; k < 8; ++k) mma_e(d + (uint32_t)(mode - 10) * 32u, a + 2ull * (k & 1), bd + 2ull * (k & 1), idesc);
      } else {  // the fused kernel's pattern: per dw (A shifted), per K step, N=64 at block b + N=32 at block 0
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          const uint64_t ak = a + 4ull * (k >> 1) + 2ull * (k & 1);
          mma_e(d + 64, ak, bd + 2ull * (k & 1), make_idesc_bf16(64));
          mma_e(d, ak, bd + 256 + 2ull * (k & 1), make_idesc_bf16(32));
        }
      }
    }
    if (threadIdx.x == 0) {
      commit(smem_u32(&bar));
      mbar_wait(smem_u32(&bar), 0);
      if (blockIdx.x == 0) out[0] = clock64() - t0;
      stop_flag = 1;
    }
    __syncwarp();
  } else if (inter > 0) {
    // interference warps 1..3 (TMEM lane quadrants 1..3) until the MMA warp is done:
    // 1 = tcgen05.ld 16 columns + wait, 2 = st.shared 16 B per lane, 3 = tcgen05.st 8 zero columns
    // + wait, 4 = ld.shared 16 B per lane, 5 = 1 + 2 (an epilogue's mix)
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    if (inter == 8 || inter == 9) {  // warp 1: bulk copies global -> shared (8: 16 KB, 9: 4 KB per copy) into scratch
      __shared__ __align__(8) uint64_t cbar;
      const uint32_t bytes = inter == 8 ? 16384u : 4096u;
      if (w == 1) {
        const uint32_t b = smem_u32(&cbar);
        if (ln == 0) {
          asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
          asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        uint32_t ph = 0;
        long long nb = 0;
        while (!stop_flag) {
          if (ln == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(base + 100u * 1024u - 16384u + 0u), "l"(gsrc + (nb & 63) * 1024), "r"(bytes), "r"(b) : "memory");
            asm volatile("{\n\t.reg .pred p;\nWC_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WC_%=;\n}\n" ::"r"(b), "r"(ph) : "memory");
          }
          __syncwarp();
          ph ^= 1u;
          ++nb;
        }
        if (ln == 0 && blockIdx.x == 0) out[1] = nb;
      }
      return;
    }
    if (inter == 6 || inter == 7) {  // 6: warps 4, 8, 12 (the MMA warp's scheduler) run FMA / SFU math; 7: the other warps do
      const bool busy = inter == 6 ? (w % 4 == 0) : (w % 4 != 0);
      float x = (float)ln * 1e-3f, y = 1.f;
      while (busy && !stop_flag) {
#pragma unroll 16
        for (int r = 0; r < 64; ++r) {
          x = fmaf(x, 0.999f, 1e-4f);
          float e;
          asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-x));
          y = fmaf(y, e, x);
        }
      }
      if (y == 12345.f) out[1] = 1;
      return;
    }
    if (inter == 10 && w < 4) return;  // 10: warps 4..19 (every scheduler, 16 warps) run the mix of 5 plus TMEM stores
    const uint32_t ta = tmem + ((uint32_t)((w & 3) * 32) << 16) + 256u + (uint32_t)((w >> 2) & 3) * 64u;
    const uint32_t sa = base + 96u * 1024u + (uint32_t)(w & 7) * 512u + (uint32_t)ln * 16u;
    uint32_t acc = 0;
    while (!stop_flag) {
      for (int r = 0; r < 16; ++r) {
        if (inter == 1 || inter == 5 || inter == 10) {
          uint32_t v[16];
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                       : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                         "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                       : "r"(ta));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          for (int e = 0; e < 16; ++e) acc += v[e];
        }
        if (inter == 2 || inter == 5 || inter == 10)
          asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(sa), "r"(acc) : "memory");
        if (inter == 3 || inter == 10) {
          asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(ta), "r"(0u) : "memory");
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        if (inter == 4) {
          uint32_t a0, a1, a2, a3;
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "r"(sa));
          acc += a0 ^ a1 ^ a2 ^ a3;
        }
      }
    }
    if (acc == 0x12345678u) out[1] = acc;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  uint4* gsrc;
  cudaMalloc(&gsrc, 64 * 16384 + 16384);
  cudaMemset(gsrc, 0, 64 * 16384 + 16384);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024 + 4096);
  struct Case { int layout, n, shift, rotD, rotA; uint32_t data; int mode; int inter; int sboA; } cases[] = {
      // halo-tile A operands: core groups (Wt + 2) rows apart (SW128: 1280 B, SW64: 640 B), starts shifted by 0..2 rows
      {2, 192, 0, 0, 1, 1u, 0, 0, 0}, {2, 160, 0, 0, 1, 1u, 0, 0, 0}, {2, 224, 0, 0, 1, 1u, 0, 0, 0},
      {2, 256, 0, 0, 1, 1u, 0, 0, 0}, {2, 128, 0, 0, 1, 1u, 0, 0, 0}, {2, 64, 0, 0, 1, 1u, 0, 0, 0},
      {4, 96, 0, 0, 1, 1u, 0, 10, 0}, {4, 96, 0, 0, 1, 1u, 4, 10, 0}, {2, 128, 0, 0, 1, 1u, 0, 10, 0},
      {2, 128, 0, 0, 1, 1u, 0, 8, 0}, {2, 128, 0, 0, 1, 1u, 0, 9, 0}, {4, 96, 0, 0, 1, 1u, 0, 8, 0}, {4, 64, 0, 0, 1, 1u, 0, 8, 0},
      {2, 128, 0, 0, 1, 1u, 0, 0, 0}, {2, 128, 0, 0, 1, 1u, 0, 0, 1280}, {2, 128, 1, 0, 1, 1u, 0, 0, 1280},
      {2, 128, 2, 0, 1, 1u, 0, 0, 1280}, {2, 64, 0, 0, 1, 1u, 0, 0, 0}, {2, 64, 1, 0, 1, 1u, 0, 0, 1280},
      {4, 32, 0, 0, 1, 1u, 0, 0, 0}, {4, 32, 1, 0, 1, 1u, 0, 0, 640}, {4, 96, 1, 0, 1, 1u, 0, 0, 640},
      // concurrent traffic from 3 other warps (inter 1..5) during N = 96 / 128 MMAs, D fixed (columns 0..N-1)
      {4, 96, 0, 0, 1, 1u, 0, 0}, {4, 96, 0, 0, 1, 1u, 0, 1}, {4, 96, 0, 0, 1, 1u, 0, 2}, {4, 96, 0, 0, 1, 1u, 0, 3},
      {4, 96, 0, 0, 1, 1u, 0, 4}, {4, 96, 0, 0, 1, 1u, 0, 5}, {4, 96, 0, 0, 1, 1u, 4, 0}, {4, 96, 0, 0, 1, 1u, 4, 5},
      {2, 128, 0, 0, 1, 1u, 0, 0}, {2, 128, 0, 0, 1, 1u, 0, 1}, {2, 128, 0, 0, 1, 1u, 0, 2}, {2, 128, 0, 0, 1, 1u, 0, 5},
      {4, 96, 0, 0, 1, 1u, 0, 6}, {4, 96, 0, 0, 1, 1u, 0, 7}, {4, 96, 0, 0, 1, 1u, 4, 6}, {2, 128, 0, 0, 1, 1u, 0, 6},
      {4, 96, 0, 1, 1, 1u, 0}, {4, 96, 0, 1, 1, 1u, 4}, {4, 96, 0, 1, 1, 1u, 5}, {4, 96, 0, 1, 1, 1u, 0},
      {4, 96, 0, 1, 1, 1u, 10}, {4, 96, 0, 1, 1, 1u, 11}, {4, 96, 0, 0, 1, 1u, 12}, {4, 96, 0, 0, 1, 1u, 13},
      {4, 64, 0, 1, 1, 1u, 10}, {4, 64, 0, 1, 1, 1u, 11}, {4, 64, 0, 1, 1, 1u, 12}, {4, 64, 0, 0, 1, 1u, 13},
      {4, 32, 0, 1, 1, 1u, 10}, {4, 32, 0, 1, 1, 1u, 11}, {4, 32, 0, 1, 1, 1u, 13},
      {4, 96, 0, 1, 1, 1u, 1}, {4, 96, 0, 1, 1, 1u, 2}, {4, 96, 0, 1, 1, 1u, 3},
      {4, 32, 0, 1, 1, 1u}, {4, 96, 0, 1, 1, 1u}, {4, 64, 0, 1, 1, 1u}, {4, 128, 0, 1, 1, 1u}, {4, 256, 0, 1, 1, 1u},
      {4, 32, 0, 0, 0, 0u},          {4, 32, 0, 0, 0, 0x3c003c00u}, {4, 96, 0, 0, 0, 0u},
      {4, 96, 0, 0, 0, 0x3c003c00u}, {4, 96, 0, 1, 0, 0x3c003c00u}, {4, 96, 0, 0, 1, 0x3c003c00u},
      {4, 96, 1, 0, 0, 0x3c003c00u}, {4, 32, 0, 1, 1, 0x3c003c00u}, {4, 64, 0, 1, 1, 0x3c003c00u},
      {4, 128, 0, 1, 1, 0x3c003c00u}, {4, 256, 0, 1, 1, 0x3c003c00u}, {2, 32, 0, 1, 1, 0x3c003c00u},
      {2, 64, 0, 1, 1, 0x3c003c00u}, {2, 96, 0, 1, 1, 0x3c003c00u}, {2, 128, 0, 1, 1, 0x3c003c00u},
      {2, 256, 0, 1, 1, 0x3c003c00u},
  };
  for (auto& c : cases) {
    for (int rep = 0; rep < 2; ++rep) {
      probe<<<148, c.inter == 10 ? 640 : (c.inter == 6 || c.inter == 7) ? 512 : 128, 100 * 1024 + 4096>>>(c.layout, c.n, c.shift, c.rotD, c.rotA, c.data, c.mode, c.inter, c.sboA, gsrc, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error: %s\n", cudaGetErrorString(e)); return 1; }
    }
    long long clk, nb = 0;
    cudaMemcpy(&clk, d, 8, cudaMemcpyDeviceToHost);
    if (c.inter == 8 || c.inter == 9) cudaMemcpy(&nb, d + 1, 8, cudaMemcpyDeviceToHost);
    if (nb) printf("  (bulk copies during the run: %lld, %.1f B/clk)\n", nb, (double)nb * (c.inter == 8 ? 16384 : 4096) / clk);
    const double per = (double)clk / (NIT * (c.mode == 3 ? 12 : (c.mode == 4 || c.mode == 5) ? 6 : 8));
    printf("sboA %4d mode %d inter %d %s N=%3d shift=%d rotD=%d rotA=%d data=%s : %6.1f clk/MMA (tensor floor %5.1f), operand B/clk %6.1f\n",
           c.sboA, c.mode, c.inter, c.layout == 4 ? "SW64 " : "SW128", c.n, c.shift, c.rotD, c.rotA, c.data == 1u ? "rand " : c.data ? "1/128" : "zero ", per, c.n / 2.0,
           (128.0 * 32 + c.n * 32.0) / per);
  }
  return 0;
}
