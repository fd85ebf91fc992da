// Residency probe of the fused head kernel: what the runtime's occupancy calculator and the
// function attributes say for img2feat_tc_kernel<32/64> (tools only; includes the product TU).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o tools/occ_probe tools/occ_probe.cu -lcuda
#include "../paper_2605_19705_b200/csrc/conv_tc.cu"
#include <cstdio>
namespace ideq { bool pdl_enabled() { return false; } }
template <typename K>
static void probe(const char* name, K k) {
  int o = -1;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, 128, 0);
  cudaFuncAttributes a;
  cudaError_t e2 = cudaFuncGetAttributes(&a, k);
  printf("%s: occupancy api -> %d (%s); attrs (%s): static smem %zu, regs %d, maxDyn %d, maxThreads %d\n", name, o,
         cudaGetErrorString(e), cudaGetErrorString(e2), a.sharedSizeBytes, a.numRegs, a.maxDynamicSharedSizeBytes,
         a.maxThreadsPerBlock);
  for (int carve : {-1, 100}) {
    if (carve >= 0) cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, 128, 0);
    printf("   carveout %d -> %d (%s)\n", carve, o, cudaGetErrorString(e));
  }
}
int main() {
  cudaSetDevice(0);
  cudaFree(0);
  int smsm = 0, res = 0;
  cudaDeviceGetAttribute(&smsm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, 0);
  cudaDeviceGetAttribute(&res, cudaDevAttrReservedSharedMemoryPerBlock, 0);
  printf("smem per SM %d, reserved per block %d\n", smsm, res);
  probe("img2feat<32>", ideq::img2feat_tc_kernel<32>);
  probe("img2feat<64>", ideq::img2feat_tc_kernel<64>);
  return 0;
}
