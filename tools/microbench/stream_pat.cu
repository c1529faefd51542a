// Streaming pattern of the lane-range design (no HMM math): every lane owns a contiguous range of n
// steps (16 B each) and walks it in slices of S steps with per-lane bulk copies.
//   pass A: loads only (3-stage ring), a trivial reduction per row
//   pass B: load + two per-lane bulk stores (filtered / smoothed) per slice (2-stage ring + out buffer)
// Reports achieved GB/s for T = 1e8 steps.
#include <cstdio>
#include <cstdint>
#include "../../paper_2102_05743_b200/csrc/hmm_device.cuh"
using namespace hmm;

#ifndef NT_
#define NT_ 256
#define S_ 16
#endif
constexpr int NT = NT_, S = S_, SB = S * 16, PITCH = SB + 16;

__global__ void __launch_bounds__(NT) passA(const float4* ll, int64_t T, int64_t n, float* sink, int NS) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar[4][NT / 32];
    const int tid = threadIdx.x, w = tid >> 5;
    if (tid < 32) for (int s = 0; s < NS; s++) if (tid == 0) for (int q = 0; q < NT / 32; q++) mbar_init(&bar[s][q], 32);
    if (tid == 0) fence_mbar_init();
    __syncthreads();
    const int64_t g = (int64_t)blockIdx.x * NT + tid;
    int64_t a = g * n, e = a + n; if (e > T) e = T;
    const int K = a < e ? (int)((e - a + S - 1) / S) : 0;
    const int Kmax = (int)(n / S);
    auto issue = [&](int k) {
        int s = k % NS;
        int64_t r0 = a + (int64_t)k * S;
        int rows = (k < K) ? (int)((e - r0 < S) ? e - r0 : S) : 0;
        uint32_t bytes = rows * 16;
        mbar_arrive_expect_tx(&bar[s][w], bytes);
        if (bytes) bulk_g2s(sm + (size_t)s * NT * PITCH + (size_t)tid * PITCH, ll + r0, bytes, &bar[s][w]);
    };
    float acc = 0.f;
    for (int k = 0; k < NS - 1 && k < Kmax; k++) issue(k);
    for (int k = 0; k < Kmax; k++) {
        if (k + NS - 1 < Kmax) issue(k + NS - 1);
        int s = k % NS;
        mbar_wait(&bar[s][w], (k / NS) & 1);
        const float4* rows = reinterpret_cast<const float4*>(sm + (size_t)s * NT * PITCH + (size_t)tid * PITCH);
        int64_t r0 = a + (int64_t)k * S;
        int nr = (k < K) ? (int)((e - r0 < S) ? e - r0 : S) : 0;
        for (int i = 0; i < nr; i++) { float4 v = rows[i]; acc += v.x * v.y + v.z * v.w; }
        __syncwarp();
    }
    if (acc == 12345.f) sink[0] = acc;
}

__global__ void __launch_bounds__(NT) passB(const float4* ll, float4* o1, float4* o2, int64_t T, int64_t n) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar[2][NT / 32];
    const int tid = threadIdx.x, w = tid >> 5;
    if (tid == 0) { for (int s = 0; s < 2; s++) for (int q = 0; q < NT / 32; q++) mbar_init(&bar[s][q], 32); fence_mbar_init(); }
    __syncthreads();
    uint8_t* fbuf = sm + 2 * (size_t)NT * PITCH;
    const int64_t g = (int64_t)blockIdx.x * NT + tid;
    int64_t a = g * n, e = a + n; if (e > T) e = T;
    const int K = a < e ? (int)((e - a + S - 1) / S) : 0;
    const int Kmax = (int)(n / S);
    auto rows_of = [&](int k) { int64_t r0 = a + (int64_t)k * S; return (k < K) ? (int)((e - r0 < S) ? e - r0 : S) : 0; };
    auto issue = [&](int k) {
        int s = k & 1;
        uint32_t bytes = rows_of(k) * 16;
        mbar_arrive_expect_tx(&bar[s][w], bytes);
        if (bytes) bulk_g2s(sm + (size_t)s * NT * PITCH + (size_t)tid * PITCH, ll + a + (int64_t)k * S, bytes, &bar[s][w]);
    };
    if (Kmax > 0) issue(0);
    for (int k = 0; k < Kmax; k++) {
        bulk_wait_read_all();             // previous slice's stores have read smem
        if (k + 1 < Kmax) issue(k + 1);
        int s = k & 1;
        mbar_wait(&bar[s][w], (k >> 1) & 1);
        float4* rows = reinterpret_cast<float4*>(sm + (size_t)s * NT * PITCH + (size_t)tid * PITCH);
        float4* f = reinterpret_cast<float4*>(fbuf + (size_t)tid * PITCH);
        int nr = rows_of(k);
        for (int i = 0; i < nr; i++) { float4 v = rows[i]; f[i] = make_float4(v.y, v.x, v.w, v.z); rows[i] = make_float4(v.w, v.z, v.y, v.x); }
        fence_proxy_async_smem();
        if (nr) {
            bulk_s2g(o1 + a + (int64_t)k * S, f, nr * 16);
            bulk_s2g(o2 + a + (int64_t)k * S, rows, nr * 16);
            bulk_commit();
        }
    }
    bulk_wait_all();
}

int main() {
    const int64_t T = 100000000;
    const int G = 148;
    const int64_t L = (int64_t)G * NT;
    int64_t n = (T + L - 1) / L; n = (n + S - 1) / S * S;
    float4 *ll, *o1, *o2; float* sink;
    cudaMalloc(&ll, T * 16); cudaMalloc(&o1, T * 16); cudaMalloc(&o2, T * 16); cudaMalloc(&sink, 4);
    cudaMemset(ll, 0, T * 16);
    size_t smA = 3 * (size_t)NT * PITCH, smB = 3 * (size_t)NT * PITCH;
    cudaFuncSetAttribute(passA, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smA);
    cudaFuncSetAttribute(passB, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smB);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int NS : {2, 3}) {
        float best = 1e9;
        for (int r = 0; r < 5; r++) {
            cudaEventRecord(e0); passA<<<G, NT, NS * (size_t)NT * PITCH>>>(ll, T, n, sink, NS); cudaEventRecord(e1);
            cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
        }
        printf("passA NS=%d: %.3f ms  %.0f GB/s read  (%s)\n", NS, best, T * 16 / (best * 1e6), cudaGetErrorString(cudaGetLastError()));
    }
    {
        float best = 1e9;
        for (int r = 0; r < 5; r++) {
            cudaEventRecord(e0); passB<<<G, NT, smB>>>(ll, o1, o2, T, n); cudaEventRecord(e1);
            cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
        }
        printf("passB: %.3f ms  %.0f GB/s (r+w)  (%s)\n", best, T * 48 / (best * 1e6), cudaGetErrorString(cudaGetLastError()));
    }
    {   // reference: plain copy kernel bandwidth via cudaMemcpy D2D
        float best = 1e9;
        for (int r = 0; r < 5; r++) {
            cudaEventRecord(e0); cudaMemcpyAsync(o1, ll, T * 16, cudaMemcpyDeviceToDevice); cudaEventRecord(e1);
            cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
        }
        printf("memcpy D2D 1.6 GB: %.3f ms  %.0f GB/s (r+w)\n", best, T * 32 / (best * 1e6));
    }
    return 0;
}
