// Launch cost of an empty 148-CTA kernel: regular vs cooperative launch (cudaLaunchKernelEx with
// cudaLaunchAttributeCooperative), device time between events on one stream, 229 KB dynamic SMEM.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void empty_kernel(int* p) { if (p && threadIdx.x == 0 && blockIdx.x == 1000000) p[0] = 1; }
int main() {
    const size_t smem = 229888;
    cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaStream_t s; cudaStreamCreate(&s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int coop = 0; coop < 2; coop++) {
        for (int rep = 0; rep < 2; rep++) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(148); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = smem; cfg.stream = s;
            cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeCooperative; a[0].val.cooperative = 1;
            cfg.attrs = a; cfg.numAttrs = coop;
            const int N = 200;
            cudaEventRecord(e0, s);
            for (int i = 0; i < N; i++) cudaLaunchKernelEx(&cfg, empty_kernel, (int*)nullptr);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (rep) printf("%s launch: %.2f us per kernel (back to back, %d launches)\n", coop ? "cooperative" : "regular", ms * 1e3 / N, N);
        }
    }
    return 0;
}
