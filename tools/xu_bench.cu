// Microbenchmark: per-SM throughput of the epilogue's candidate instructions on B200
// (ex2.approx on MUFU, cvt.rn.bf16x2.f32 pack, an FMA-pipe polynomial exp2, R2UR-free FFMA).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xu_bench tools/xu_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ float exp2_poly(float x) {  // x <= 0, FMA/ALU only
  x = fmaxf(x, -126.f);
  const float j = x + 12582912.f;               // round to nearest integer in the mantissa
  const float n = j - 12582912.f;
  const float f = x - n;                        // [-0.5, 0.5]
  float p = 1.3333558146428443e-3f;
  p = fmaf(p, f, 9.6181291076284772e-3f);
  p = fmaf(p, f, 5.5504108664821580e-2f);
  p = fmaf(p, f, 2.4022650695910071e-1f);
  p = fmaf(p, f, 6.9314718055994531e-1f);
  p = fmaf(p, f, 1.f);
  return __int_as_float(__float_as_int(p) + ((__float_as_int(j) - 0x4B400000) << 23));
}

template <int OP>
__global__ void __launch_bounds__(256) bench(float* out, int iters, long long* cyc) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  uint32_t acc = 0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) a[i] = exp2f(a[i]) - 1.0f;                     // MUFU.EX2
      if (OP == 1) {                                             // F2FP pack
        __nv_bfloat162 h = __floats2bfloat162_rn(a[i], a[(i + 1) & 7]);
        acc += *reinterpret_cast<uint32_t*>(&h);
        a[i] += 1e-7f;
      }
      if (OP == 2) a[i] = exp2_poly(a[i]) - 1.0f;                // FMA poly
      if (OP == 3) a[i] = fmaf(a[i], 0.999f, -1e-4f);            // plain FFMA
    }
  }
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* d;
  long long* c;
  cudaMalloc(&d, 148 * 8 * 256 * 4);
  cudaMalloc(&c, 148 * 8 * 8);
  const int iters = 4096;
  const char* names[4] = {"ex2.approx (MUFU)", "cvt bf16x2 pack (F2FP)", "exp2 FMA polynomial", "FFMA"};
  for (int op = 0; op < 4; ++op) {
    for (int bps : {4, 8}) {
      const int grid = 148 * bps;
      if (op == 0) bench<0><<<grid, 256>>>(d, iters, c);
      if (op == 1) bench<1><<<grid, 256>>>(d, iters, c);
      if (op == 2) bench<2><<<grid, 256>>>(d, iters, c);
      if (op == 3) bench<3><<<grid, 256>>>(d, iters, c);
      cudaDeviceSynchronize();
      long long h[148 * 8];
      cudaMemcpy(h, c, grid * 8, cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
      // ops per SM during the (max) block time: bps blocks x 256 threads x iters x 8
      const double ops = (double)bps * 256 * iters * 8;
      printf("%-26s blocks/SM=%d : %.1f results/clk/SM\n", names[op], bps, ops / mx);
    }
  }
  return 0;
}
