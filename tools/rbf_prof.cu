// Stage timeline of the fused residual-block kernel (CTA 0): builds rbf.cu with RBF_TRACE=1.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -rdc=true -DRBF_TRACE=1 -I include
//        -o tools/rbf_prof tools/rbf_prof.cu paper_2605_19705_b200/csrc/rbf.cu -lcuda
// Run:   tools/rbf_prof [vjp]
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "../paper_2605_19705_b200/csrc/kernels.h"
namespace ideq {
extern __device__ long long g_rbf_trace[16][256];
}
int main(int argc, char** argv) {
  const bool vjp = argc > 1 && atoi(argv[1]) != 0;
  const int N = 32, H = 256, W = 256, C = 32;
  const size_t n = (size_t)N * H * W * C;
  std::vector<__nv_bfloat16> hx(n), hw(9 * 32 * 32);
  srand(1);
  for (auto& v : hx) v = __float2bfloat16((rand() / (float)RAND_MAX) - 0.5f);
  for (auto& v : hw) v = __float2bfloat16(((rand() / (float)RAND_MAX) - 0.5f) * 0.1f);
  __nv_bfloat16 *x, *out, *act, *w;
  cudaMalloc(&x, n * 2); cudaMalloc(&out, n * 2); cudaMalloc(&act, n * 2); cudaMalloc(&w, hw.size() * 2);
  cudaMemcpy(x, hx.data(), n * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(act, hx.data(), n * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(w, hw.data(), hw.size() * 2, cudaMemcpyHostToDevice);
  int dh[9], dw[9];
  for (int t = 0; t < 9; ++t) { dh[t] = t / 3 - 1; dw[t] = t % 3 - 1; }
  ideq::init_attrs_rbf();
  char err[256];
  ideq::RbfPlan* p = ideq::rbf_make_plan(vjp, N, H, W, dh, dw, dh, dw, w, w, x, out, act, 148, err, sizeof(err));
  if (!p) { printf("plan: %s\n", err); return 1; }
  for (int rep = 0; rep < 3; ++rep) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    ideq::rbf_launch(p, 0);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("launch %d: %.1f us\n", rep, ms * 1000);
  }
  static long long tr[16][256];
  cudaMemcpyFromSymbol(tr, ideq::g_rbf_trace, sizeof(tr));
  const long long t0 = tr[2][0];
  // per row r: S1 begin/issue (k = r), E1 begin/ready/end (iu = r), S2 begin/issue (j = r), E2 begin/ready/end (io = r)
  printf("  r   S1beg  S1iss |  E1beg  E1rdy  E1end |  S2beg  S2iss |  E2beg  E2rdy  E2end\n");
  for (int r = 16; r < 28; ++r)
    printf("%3d %7lld %6lld | %6lld %6lld %6lld | %6lld %6lld | %6lld %6lld %6lld\n", r, tr[2][r] - t0, tr[4][r] - t0,
           tr[8][r] - t0, tr[9][r] - t0, tr[10][r] - t0, tr[5][r] - t0, tr[7][r] - t0, tr[11][r] - t0, tr[12][r] - t0,
           tr[13][r] - t0);
  printf("period (E2 end, rows 10..50): %.0f clk\n", (double)(tr[13][50] - tr[13][10]) / 40);
  return 0;
}
