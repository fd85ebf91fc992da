// Stage profile of the C1 whole-solve kernel: builds tiny_solve.cu with TS_PROF=1 and prints the
// clock cycles per iteration spent in each stage (CTA 0, thread 0).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -rdc=true -DTS_PROF=1 -I include
//        -o tools/tiny_prof tools/tiny_prof.cu paper_2605_19705_b200/csrc/tiny_solve.cu
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2605_19705_b200/csrc/kernels.h"
namespace ideq { extern __device__ long long ts_prof[16]; }
namespace ideq { bool pdl_enabled() { return false; } }
int main() {
  const int H = 32, W = 32, ks = 9, K = 100;
  std::vector<float> w(16 * 9 + 16 * 16 * 9 + 16 * 9, 0.01f), k(ks * ks, 1.f / 81), y(H * W, 0.5f), x(H * W, 0.5f);
  float *dw, *dk, *dy, *dx, *dres, *dtr; int *dit, *dst, *dkd;
  cudaMalloc(&dw, w.size() * 4); cudaMalloc(&dk, k.size() * 4); cudaMalloc(&dy, y.size() * 4); cudaMalloc(&dx, x.size() * 4);
  cudaMalloc(&dres, 4); cudaMalloc(&dtr, K * 4); cudaMalloc(&dit, 4); cudaMalloc(&dst, 4); cudaMalloc(&dkd, 4);
  cudaMemcpy(dw, w.data(), w.size() * 4, cudaMemcpyHostToDevice); cudaMemcpy(dk, k.data(), k.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dy, y.data(), y.size() * 4, cudaMemcpyHostToDevice); cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
  ideq::init_attrs_tiny();
  ideq::TinySolveArgs a{};
  a.N = 1; a.H = H; a.W = W; a.ks = ks; a.kper = 0; a.kern = dk; a.w1 = dw; a.w2 = dw + 144; a.w3 = dw + 144 + 2304;
  a.y = dy; a.x = dx; a.lam = 0.05f; a.tau = 1.f; a.beta = 0.5f; a.tol = 0.f; a.max_iter = K; a.check_every = 1;
  a.iters = dit; a.res = dres; a.status = dst; a.trace = dtr; a.trace_cap = K; a.kdone = dkd;
  for (int rep = 0; rep < 2; ++rep) {
    long long zero[16] = {0};
    cudaMemcpyToSymbol(ideq::ts_prof, zero, sizeof(zero));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    ideq::launch_tiny_solve(a, 0);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long p[16]; cudaMemcpyFromSymbol(p, ideq::ts_prof, sizeof(p));
    const char* names[16] = {"(loop top)", "[1] c1+Az", "S1 sync", "[2] c2", "S2 sync", "[3,4] c3,c3T+ATr", "S3 sync", "[5] c2T", "S4 sync", "[6] c1T+upd", "S5 sync (+z)", "accept", "", "", "", ""};
    printf("total %.1f us per iteration\n", 1000.0 * ms / K);
    for (int i = 0; i < 12; ++i) printf("  %-16s %7.0f clk/iter\n", names[i], (double)p[i] / K);
  }
  return 0;
}
