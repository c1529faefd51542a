// Probe of the tcgen05 TF32 path used by the large-D leaf kernel: D[128x64] = A[128x64] . B[64x64]^T with
// A, B K-major in SMEM (SWIZZLE_NONE core matrices: 8 rows x 16 B; LBO = 128 B between K chunks,
// SBO = 2048 B between 8-row groups), D in TMEM, read back with tcgen05.ld.32x32b.x64.  Checks 1xTF32
// and 3xTF32 (hi/lo split) against an fp64 host product.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <random>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// byte offset of element (row r, k) in the K-major no-swizzle canonical layout (K = 64 tf32 per row)
__host__ __device__ inline uint32_t cm_off(int r, int k) {
    return (uint32_t)((r >> 3) * 2048 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
}
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3fff);
    d |= (uint64_t)((128 >> 4) & 0x3fff) << 16;   // LBO
    d |= (uint64_t)((2048 >> 4) & 0x3fff) << 32;  // SBO
    d |= (uint64_t)1 << 46;                        // version (sm100)
    return d;                                      // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE
}
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t dtmem, uint64_t ad, uint64_t bd, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dtmem),
        "l"(ad), "l"(bd), "r"(IDESC), "r"(acc));
}

__global__ void probe(const float* A, const float* B, float* D, int mode) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* sAh = sm;            // 32 KB
    uint8_t* sAl = sm + 32768;    // 32 KB
    uint8_t* sBh = sm + 65536;    // 16 KB
    uint8_t* sBl = sm + 81920;    // 16 KB
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 128 * 64; i += blockDim.x) {
        const int r = i / 64, k = i % 64;
        const float x = A[i];
        const float hi = __uint_as_float(__float_as_uint(x) & 0xffffe000u);
        *reinterpret_cast<float*>(sAh + cm_off(r, k)) = hi;
        *reinterpret_cast<float*>(sAl + cm_off(r, k)) = x - hi;
    }
    for (int i = tid; i < 64 * 64; i += blockDim.x) {
        const int r = i / 64, k = i % 64;
        const float x = B[i];
        const float hi = __uint_as_float(__float_as_uint(x) & 0xffffe000u);
        *reinterpret_cast<float*>(sBh + cm_off(r, k)) = hi;
        *reinterpret_cast<float*>(sBl + cm_off(r, k)) = x - hi;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    if (tid == 0) {
        const uint32_t ah = smem_u32(sAh), al = smem_u32(sAl), bh = smem_u32(sBh), bl = smem_u32(sBl);
        int n = 0;
        for (int k = 0; k < 8; k++) {  // K = 8 tf32 per instruction = 2 chunks = 256 B
            mma_tf32(tm, make_desc(ah + 256 * k), make_desc(bh + 256 * k), n++ > 0);
            if (mode == 3) {
                mma_tf32(tm, make_desc(ah + 256 * k), make_desc(bl + 256 * k), 1);
                mma_tf32(tm, make_desc(al + 256 * k), make_desc(bh + 256 * k), 1);
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
    }
    // wait for the MMAs
    {
        uint32_t done = 0;
        while (!done) {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                         : "=r"(done) : "r"(smem_u32(&mbar)));
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp < 4) {
        uint32_t v[64];
        const uint32_t taddr = tm + ((uint32_t)(warp * 32) << 16);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,"
            "%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]),
              "=r"(v[32]), "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]), "=r"(v[38]), "=r"(v[39]),
              "=r"(v[40]), "=r"(v[41]), "=r"(v[42]), "=r"(v[43]), "=r"(v[44]), "=r"(v[45]), "=r"(v[46]), "=r"(v[47]),
              "=r"(v[48]), "=r"(v[49]), "=r"(v[50]), "=r"(v[51]), "=r"(v[52]), "=r"(v[53]), "=r"(v[54]), "=r"(v[55]),
              "=r"(v[56]), "=r"(v[57]), "=r"(v[58]), "=r"(v[59]), "=r"(v[60]), "=r"(v[61]), "=r"(v[62]), "=r"(v[63])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        const int r = warp * 32 + lane;
        for (int j = 0; j < 64; j++) D[r * 64 + j] = __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tm));
}

int main() {
    std::mt19937 g(1);
    std::uniform_real_distribution<float> U(0.f, 1.f);
    std::vector<float> A(128 * 64), B(64 * 64), D(128 * 64);
    for (auto& x : A) x = U(g);
    for (auto& x : B) x = U(g);
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304 + 1024);
    for (int mode : {1, 3}) {
        cudaMemset(dD, 0, D.size() * 4);
        probe<<<1, 128, 98304 + 1024>>>(dA, dB, dD, mode);
        cudaError_t e = cudaDeviceSynchronize();
        printf("mode %d: %s\n", mode, cudaGetErrorString(e));
        if (e) return 1;
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double maxrel = 0;
        for (int r = 0; r < 128; r++)
            for (int n = 0; n < 64; n++) {
                double ref = 0;
                for (int k = 0; k < 64; k++) ref += (double)A[r * 64 + k] * (double)B[n * 64 + k];
                maxrel = fmax(maxrel, fabs(D[r * 64 + n] - ref) / fabs(ref));
            }
        printf("  max rel err vs fp64: %.3e  (D[0][0]=%f)\n", maxrel, D[0]);
    }
    return 0;
}
