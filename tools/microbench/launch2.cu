// Event vs launch overhead: N back-to-back empty kernels between one event pair (after a long fill).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void empty_k(int* p) { if (threadIdx.x == 0 && p) p[blockIdx.x] = 0; }
__global__ void fill_k(float* p, size_t n) { for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = 0.f; }
int main() {
  float* buf; size_t n = 256 << 20; cudaMalloc(&buf, n * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int N : {1, 2, 4, 16, 64}) for (int coop : {0, 1}) {
    float best = 1e9;
    for (int r = 0; r < 10; r++) {
      fill_k<<<592, 512>>>(buf, n);
      cudaEventRecord(e0);
      for (int i = 0; i < N; i++) {
        cudaLaunchConfig_t cfg = {}; cfg.gridDim = 148; cfg.blockDim = 256;
        cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeCooperative; a[0].val.cooperative = 1;
        cfg.attrs = a; cfg.numAttrs = coop; int* np = nullptr;
        cudaLaunchKernelEx(&cfg, empty_k, np);
      }
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("N %3d coop %d : total %.2f us, per kernel %.2f us\n", N, coop, 1e3 * best, 1e3 * best / N);
  }
  return 0;
}
