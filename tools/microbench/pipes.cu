// Pipe-throughput microbenchmark for sm_100a: FFMA, FFMA2, FADD2, FMNMX3, DADD, MUFU.EX2.
// Used once to size the D=4 kernels.
#include <cstdio>
#include <cuda_runtime.h>
#define N_ITER 4096
template<int OP> __global__ void kern(float* out, float a, float b) {
  float x[8]; float2 y[8]; double z[8];
  #pragma unroll
  for (int i = 0; i < 8; i++) { x[i] = threadIdx.x * 1e-3f + i; y[i] = make_float2(x[i], x[i]+1); z[i] = x[i]; }
  for (int it = 0; it < N_ITER; it++) {
    #pragma unroll
    for (int i = 0; i < 8; i++) {
      if (OP == 0) x[i] = fmaf(x[i], a, x[(i+1)&7]);             // FFMA 3-reg
      if (OP == 1) y[i] = __ffma2_rn(y[i], make_float2(a,a), y[(i+1)&7]); // FFMA2
      if (OP == 2) { float r; asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(x[i]), "f"(x[(i+1)&7]), "f"(x[(i+3)&7])); x[i] = r - a; } // FMNMX3 + FADD
      if (OP == 3) z[i] = fma(z[i], (double)a, z[(i+1)&7]);     // DFMA
      if (OP == 4) x[i] = exp2f(x[i] * a);                     // MUFU.EX2 (+FMUL)
      if (OP == 5) y[i] = __fadd2_rn(y[i], y[(i+1)&7]);         // FADD2
      if (OP == 6) x[i] = x[i] * a + b;                         // FFMA imm-ish (const operands)
      if (OP == 7) x[i] = fmaxf(x[i], x[(i+1)&7]) - a;          // FMNMX + FADD
      if (OP == 8) x[i] = x[i] + x[(i+1)&7];                    // FADD
      if (OP == 10) { y[i] = __fadd2_rn(y[i], y[(i+1)&7]); x[i] = fmaxf(x[i], x[(i+1)&7]); } // FADD2 || FMNMX
      if (OP == 11) x[i] = fmaxf(x[i], x[(i+1)&7]);             // FMNMX only
      if (OP == 9) { float r; asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(x[i]), "f"(x[(i+1)&7]), "f"(x[(i+3)&7])); x[i] = r; } // FMNMX3 only
    }
  }
  float s = 0;
  #pragma unroll
  for (int i = 0; i < 8; i++) s += x[i] + y[i].x + y[i].y + (float)z[i];
  if (s == 1234.5f) out[0] = s;
}
template<int OP> void run(const char* name, double ops_per_inner) {
  float* out; cudaMalloc(&out, 4);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  dim3 grid(nsm * 4), block(512);
  kern<OP><<<grid, block>>>(out, 0.999f, 1e-3f);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; r++) kern<OP><<<grid, block>>>(out, 0.999f, 1e-3f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double lane_ops = 5.0 * grid.x * block.x * (double)N_ITER * 8 * ops_per_inner;
  double rate = lane_ops / (ms * 1e-3);
  printf("%-10s %8.3f ms  %8.2f Tlane-op/s  %7.1f lane-op/clk/SM (at max clk %d MHz)\n", name, ms, rate / 1e12,
         rate / (nsm * clk * 1e3), clk / 1000);
}
int main() {
  run<0>("FFMA", 1); run<1>("FFMA2", 2); run<2>("FMNMX3+FADD", 2); run<3>("DFMA", 1);
  run<4>("EX2+FMUL", 2); run<5>("FADD2", 2); run<6>("FFMA-c", 1);
  run<7>("FMNMX+FADD", 2); run<8>("FADD", 1); run<9>("FMNMX3", 1);
  run<10>("FADD2||FMNMX", 3); run<11>("FMNMX", 1);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("SMs %d smemPerBlockOptin %zu smemPerSM %zu L2 %d regsPerSM %d clock %d kHz memclk %d kHz busw %d\n",
         p.multiProcessorCount, p.sharedMemPerBlockOptin, p.sharedMemPerMultiprocessor, p.l2CacheSize,
         p.regsPerMultiprocessor, p.clockRate, p.memoryClockRate, p.memoryBusWidth);
  return 0;
}
