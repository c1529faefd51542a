// Launch-overhead microbenchmark: empty kernel, 148 CTAs x 256 threads, varying dynamic SMEM,
// normal vs cooperative launch, after a memset-like kernel (carveout change) or back to back.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void empty_k(int* p) { extern __shared__ int s[]; if (threadIdx.x == 0 && p) s[0] = p[blockIdx.x]; }
__global__ void fill_k(float* p, size_t n) { for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = 0.f; }
int main() {
  float* buf; size_t n = 64 << 20; cudaMalloc(&buf, n * 4);
  cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 217440);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int smem : {0, 100000, 217440}) for (int coop : {0, 1}) for (int pre : {0, 1}) {
    float tot = 0; int reps = 20;
    for (int r = 0; r < reps + 3; r++) {
      if (pre) fill_k<<<592, 512>>>(buf, n);
      cudaEventRecord(e0);
      cudaLaunchConfig_t cfg = {}; cfg.gridDim = 148; cfg.blockDim = 256; cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeCooperative; a[0].val.cooperative = 1;
      cfg.attrs = a; cfg.numAttrs = coop; int* np = nullptr;
      cudaLaunchKernelEx(&cfg, empty_k, np);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (r >= 3) tot += ms;
    }
    printf("smem %6d coop %d after_fill %d : %.2f us per launch (event)\n", smem, coop, pre, 1e3 * tot / reps);
  }
  return 0;
}
