// Per-SM tile load of 108 KB (T=1e6 GE tile) from cold HBM: cp.async.bulk with P pieces vs LDG.128.
#include <cstdio>
#include <cstdint>
#include "../../paper_2102_05743_b200/csrc/hmm_device.cuh"
using namespace hmm;
__global__ void bulk_k(const float* g, int bytes_per_cta, int pieces, unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[64];
  if (threadIdx.x == 0) { for (int i = 0; i < pieces; i++) mbar_init(&bar[i], 1); fence_mbar_init(); }
  __syncthreads();
  unsigned long long t0 = global_ns();
  const char* src = reinterpret_cast<const char*>(g) + (size_t)blockIdx.x * bytes_per_cta;
  int pb = bytes_per_cta / pieces;
  if (threadIdx.x < pieces) {  // one issuing thread per piece
    int i = threadIdx.x;
    mbar_arrive_expect_tx(&bar[i], pb);
    bulk_g2s(sm + (size_t)i * pb, src + (size_t)i * pb, pb, &bar[i]);
  }
  if (threadIdx.x < pieces) mbar_wait(&bar[threadIdx.x], 0);
  __syncthreads();
  unsigned long long t1 = global_ns();
  if (threadIdx.x == 0) { out[2 * blockIdx.x] = t0; out[2 * blockIdx.x + 1] = t1; }
}
__global__ void ldg_k(const float4* g, int f4_per_cta, unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  float4* s = reinterpret_cast<float4*>(sm);
  unsigned long long t0 = global_ns();
  const float4* src = g + (size_t)blockIdx.x * f4_per_cta;
  #pragma unroll 8
  for (int i = threadIdx.x; i < f4_per_cta; i += blockDim.x) s[i] = __ldcs(src + i);
  __syncthreads();
  unsigned long long t1 = global_ns();
  if (threadIdx.x == 0) { out[2 * blockIdx.x] = t0; out[2 * blockIdx.x + 1] = t1; }
}
template <int K>
__global__ void ldgk_k(const float4* g, int f4_per_cta, unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  float4* s = reinterpret_cast<float4*>(sm);
  unsigned long long t0 = global_ns();
  const float4* src = g + (size_t)blockIdx.x * f4_per_cta;
  for (int base = 0; base < f4_per_cta; base += K * blockDim.x) {
    float4 r[K];
    #pragma unroll
    for (int k = 0; k < K; k++) { int i = base + k * blockDim.x + threadIdx.x; if (i < f4_per_cta) r[k] = __ldcs(src + i); }
    #pragma unroll
    for (int k = 0; k < K; k++) { int i = base + k * blockDim.x + threadIdx.x; if (i < f4_per_cta) s[i] = r[k]; }
  }
  __syncthreads();
  unsigned long long t1 = global_ns();
  if (threadIdx.x == 0) { out[2 * blockIdx.x] = t0; out[2 * blockIdx.x + 1] = t1; }
}
// every thread issues `per` bulk copies of `pb` bytes, all completing on one mbarrier per warp
__global__ void thr_bulk_k(const float* g, int bytes_per_cta, int per, unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[32];
  const int w = threadIdx.x >> 5;
  if (threadIdx.x == 0) { for (int i = 0; i < 32; i++) mbar_init(&bar[i], 32); fence_mbar_init(); }
  __syncthreads();
  unsigned long long t0 = global_ns();
  const char* src = reinterpret_cast<const char*>(g) + (size_t)blockIdx.x * bytes_per_cta;
  const int nc = blockDim.x * per;
  const int pb = (bytes_per_cta / nc) & ~15;
  mbar_arrive_expect_tx(&bar[w], pb * per);
  for (int j = 0; j < per; j++) {
    const int i = j * blockDim.x + threadIdx.x;  // interleaved so consecutive threads hit consecutive pieces
    bulk_g2s(sm + (size_t)i * pb, src + (size_t)i * pb, pb, &bar[w]);
  }
  mbar_wait(&bar[w], 0);
  __syncthreads();
  unsigned long long t1 = global_ns();
  if (threadIdx.x == 0) { out[2 * blockIdx.x] = t0; out[2 * blockIdx.x + 1] = t1; }
}
int main() {
  const int bytes = 108160; size_t total = (size_t)bytes * 148;
  float* g; cudaMalloc(&g, total + 4096); cudaMemset(g, 0, total);
  float* fl; cudaMalloc(&fl, 512 << 20);
  unsigned long long* d; cudaMalloc(&d, 8 * 2 * 148);
  cudaFuncSetAttribute(bulk_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(ldg_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  auto report = [&](const char* name) {
    unsigned long long h[296]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, t1 = 0; double mx = 0;
    if (h[0] == 0) printf("  (raw %llu %llu %s)\n", h[0], h[1], cudaGetErrorString(cudaGetLastError()));
    for (int b = 0; b < 148; b++) { t0 = h[2*b] < t0 ? h[2*b] : t0; t1 = h[2*b+1] > t1 ? h[2*b+1] : t1; double dd = (h[2*b+1]-h[2*b]); mx = dd > mx ? dd : mx; }
    printf("%-22s span %.2f us (slowest CTA %.2f us) -> %.0f GB/s aggregate\n", name, (t1 - t0) / 1e3, mx / 1e3, total / ((t1 - t0) * 1.0));
  };
  for (int pieces : {1, 2, 8, 32, 64}) {
    for (int r = 0; r < 3; r++) { cudaMemset(fl, r, 512 << 20); bulk_k<<<148, 256, bytes>>>(g, bytes - bytes % (16 * pieces), pieces, d); { cudaError_t le = cudaGetLastError(); if (le) printf("launch %s\n", cudaGetErrorString(le)); } cudaError_t e = cudaDeviceSynchronize(); if (e) printf("bulk err %s\n", cudaGetErrorString(e)); }
    char nm[64]; snprintf(nm, 64, "bulk, %d pieces", pieces); report(nm);
  }
  for (int nt : {256, 512, 1024}) {
    for (int r = 0; r < 3; r++) { cudaMemset(fl, r, 512 << 20); ldg_k<<<148, nt, bytes>>>((const float4*)g, bytes / 16, d); cudaDeviceSynchronize(); }
    char nm[64]; snprintf(nm, 64, "ldg.128 x %d threads", nt); report(nm);
  }
  cudaFuncSetAttribute(ldgk_k<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(ldgk_k<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int nt : {256, 512}) {
    for (int r = 0; r < 3; r++) { cudaMemset(fl, r, 512 << 20); ldgk_k<8><<<148, nt, bytes>>>((const float4*)g, bytes / 16, d); cudaDeviceSynchronize(); }
    char nm[64]; snprintf(nm, 64, "ldg x8 regs x %d thr", nt); report(nm);
    for (int r = 0; r < 3; r++) { cudaMemset(fl, r, 512 << 20); ldgk_k<16><<<148, nt, bytes>>>((const float4*)g, bytes / 16, d); cudaDeviceSynchronize(); }
    snprintf(nm, 64, "ldg x16 regs x %d thr", nt); report(nm);
  }
  cudaFuncSetAttribute(thr_bulk_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int nt : {256, 512}) for (int per : {1, 2, 4}) {
    for (int r = 0; r < 3; r++) { cudaMemset(fl, r, 512 << 20); thr_bulk_k<<<148, nt, bytes>>>(g, bytes, per, d); cudaError_t e = cudaDeviceSynchronize(); if (e) printf("err %s\n", cudaGetErrorString(e)); }
    char nm[64]; snprintf(nm, 64, "thr bulk %dthr x%d (%dB)", nt, per, (bytes / (nt * per)) & ~15); report(nm);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
