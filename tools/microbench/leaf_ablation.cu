// Ablation of the D=4 sum-product leaf step: which part limits cycles/step (8 and 16 warps/SM).
#include <cstdio>
#include <cstdint>
#include "../../paper_2102_05743_b200/csrc/hmm_device.cuh"
using namespace hmm;
// V: bit0 = no exp (l = v), bit1 = no renorm, bit2 = tree max, bit3 = no smem load (synthetic v)
template <int V>
__device__ __forceinline__ void leaf(const float* rows, int n, const float* A, float* P, float& sink) {
  float s = 1.0f;
  for (int i = 0; i < n; i++) {
    float v[4];
    if (V & 8) { v[0] = 0.3f * i; v[1] = v[0] + 0.1f; v[2] = v[0] - 0.2f; v[3] = v[0] + 0.05f; }
    else { float4 x = *reinterpret_cast<const float4*>(rows + i * 4); v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w; }
    float l[4];
    if (V & 1) { for (int j = 0; j < 4; j++) l[j] = v[j]; }
    else { float m = fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3])); for (int j = 0; j < 4; j++) l[j] = ex2((v[j] - m) * kLog2e); }
    float cs[4]; for (int j = 0; j < 4; j++) cs[j] = l[j] * s;
    float Q[16];
    #pragma unroll
    for (int r = 0; r < 4; r++)
      #pragma unroll
      for (int j = 0; j < 4; j++) {
        float acc = P[r * 4] * A[j];
        #pragma unroll
        for (int k = 1; k < 4; k++) acc = fmaf(P[r * 4 + k], A[k * 4 + j], acc);
        Q[r * 4 + j] = acc * cs[j];
      }
    #pragma unroll
    for (int e = 0; e < 16; e++) P[e] = Q[e];
    if (!(V & 2)) {
      float m;
      if (V & 4) {  // balanced tree of 3-input max
        float a = max3(P[0], P[1], P[2]), b = max3(P[3], P[4], P[5]), c = max3(P[6], P[7], P[8]);
        float d = max3(P[9], P[10], P[11]), e = max3(P[12], P[13], P[14]);
        m = max3(max3(a, b, c), d, fmaxf(e, P[15]));
      } else { m = vmax<16>(P); }
      s = pow2_inv(m);
    }
  }
  sink += P[0] + P[5];
}
template <int V>
__global__ void k(unsigned long long* out, int S) {
  extern __shared__ float sm[];
  for (int i = threadIdx.x; i < blockDim.x * S * 4; i += blockDim.x) sm[i] = 0.5f + 0.25f * __sinf(i * 0.37f);
  float A[16]; for (int e = 0; e < 16; e++) A[e] = 0.2f + 0.01f * e;
  __syncthreads();
  float P[16]; for (int e = 0; e < 16; e++) P[e] = (e % 5 == 0) ? 1.f : 0.1f;
  float sink = 0;
  long long t0 = clock64();
  for (int rep = 0; rep < 4; rep++) leaf<V>(sm + threadIdx.x * S * 4, S, A, P, sink);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (sink == 1234.5f) out[999] = 1;
}
template <int V> void run(const char* name, int nt) {
  unsigned long long* d; cudaMalloc(&d, 8 * 1000);
  int S = 27; size_t smem = (size_t)nt * S * 16;
  cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<V><<<148, nt, smem>>>(d, S); cudaDeviceSynchronize();
  unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-28s %2d warps: %6.1f cycles/step/warp  %5.1f SM-cycles/warp-step  %s\n", name, nt / 32, h / (4.0 * S),
         h / (4.0 * S) / (nt / 32), cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}
int main() {
  for (int nt : {256, 512}) {
    run<0>("full", nt); run<4>("full, tree max", nt); run<1>("no exp", nt); run<2>("no renorm", nt);
    run<3>("no exp, no renorm", nt); run<11>("no exp/renorm/load", nt); run<8>("no smem load", nt);
  }
  return 0;
}
