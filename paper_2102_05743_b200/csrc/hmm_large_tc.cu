// hmm_large_tc.cu — tensor-core (tcgen05, TF32x3) leaf products of the sum-product scan at D = 33..64
// (padded DP = 64), sm_100a.
//
// The leaf reduce of Algorithm 3 folds psi_t = A diag(l_t) (Eq. 5) into
// P <- P psi_t = (P A) diag(l_t).  The product P A is a dense 64x64x64 contraction with the SAME right
// operand A at every step and for every leaf, so two leaves are stacked as one M = 128 operand and
// every step is one tcgen05 MMA group  D[128x64] (TMEM) = [P_a; P_b] [128x64] . A [64x64]
// ("3xTF32 on tcgen05 at D=64 SP").  The diag(l_t) scaling, the per-row
// power-of-two renormalisation and the hi/lo split for the next step run in the epilogue:
//
//   accuracy (stated check): each fp32 operand x is split x = hi + lo with hi = x truncated to TF32 (10
//   mantissa bits) and lo = x - hi (exact); P A = Ph Ah + Ph Al + Pl Ah (the Pl Al term, ~2^-22
//   relative, is dropped) accumulated in fp32 in TMEM.  tools/microbench/tc_probe.cu measures
//   2.2e-6 max relative error per 64-term product vs fp64 (1xTF32: 8.1e-4); the parity tests run the
//   D = 33..64 configurations through this path at the 1e-5 marginal bar (tests/test_gpu_parity.py,
//   tests/test_gpu_tc.py).
//
//   rows are renormalised independently (exact pow2, exponent e_r tracked per row): the true leaf
//   product is diag(2^e) P~, so no cross-thread reduction sits on the per-step critical path; the
//   row exponents are folded back at the end of the leaf.
//
// Layout: A and B operands K-major in SMEM, SWIZZLE_NONE canonical core matrices (8 rows x 16 B),
// LBO = 128 B between K chunks, SBO = 2048 B between 8-row groups; one MMA instruction covers K = 8.
// CTA = 256 threads = 2 independent leaf pairs (warps 0-3, 4-7) ping-ponging on the tensor pipe;
// thread = one row of the stacked 128-row operand (TMEM lane = row; warp w reads lanes 32(w%4)..).
#include <cstdint>
#include <cstring>

#include "hmm_device.cuh"
#include "hmm_large.h"

namespace hmm {

namespace {

__device__ __forceinline__ uint32_t tc_off(int r, int k) {
    return (uint32_t)((r >> 3) * 2048 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
}
__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3fffu);
    d |= (uint64_t)(128u >> 4) << 16;   // leading byte offset: next K chunk
    d |= (uint64_t)(2048u >> 4) << 32;  // stride byte offset: next 8-row group
    d |= (uint64_t)1 << 46;             // descriptor version (sm_100)
    return d;                           // base offset 0, layout SWIZZLE_NONE
}
// kind::tf32, D fp32, A/B TF32 K-major, N = 64, M = 128
constexpr uint32_t kTcIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void tc_mma(uint32_t dtmem, uint64_t ad, uint64_t bd, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dtmem),
        "l"(ad), "l"(bd), "r"(kTcIdesc), "r"(acc));
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ void tmem_ld64(uint32_t taddr, float* v) {
    uint32_t r[64];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,"
        "%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
          "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
          "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
          "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
          "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 64; j++) v[j] = __uint_as_float(r[j]);
}

// Row renormalisation by an exact power of two; returns the exponent added to the row's record.
__device__ __forceinline__ int row_pow2(float* v) {
    float m = 0.0f;
#pragma unroll
    for (int j = 0; j < 64; j++) m = fmaxf(m, v[j]);
    const uint32_t E = (__float_as_uint(m) >> 23) & 0xffu;
    if (E == 0u || E >= 254u) return 0;  // zero / denormal / huge row: leave it (NaN propagates)
    const float s = __uint_as_float((254u - E) << 23);
#pragma unroll
    for (int j = 0; j < 64; j++) v[j] *= s;
    return (int)E - 127;
}
// Store a row as hi (TF32-truncated) and lo parts into the pair's K-major operand buffers.
__device__ __forceinline__ void store_split(uint8_t* Ah, uint8_t* Al, int rr, const float* v) {
#pragma unroll
    for (int k4 = 0; k4 < 64; k4 += 4) {
        float h[4], l[4];
#pragma unroll
        for (int c = 0; c < 4; c++) {
            h[c] = __uint_as_float(__float_as_uint(v[k4 + c]) & 0xffffe000u);
            l[c] = v[k4 + c] - h[c];
        }
        const uint32_t o = tc_off(rr, k4);
        *reinterpret_cast<float4*>(Ah + o) = make_float4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<float4*>(Al + o) = make_float4(l[0], l[1], l[2], l[3]);
    }
}

}  // namespace

// l_t(j) = exp(ll_t(j) - m_t) for j < D, 0 for the padding; one warp per (sequence, step) row.
__global__ void __launch_bounds__(256) lg_lik_kernel(const LgParams p, float* lik) {
    const int lane = threadIdx.x & 31;
    const int64_t rows = p.B * p.T;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t row = w0; row < rows; row += nw) {
        const float* src = p.log_lik + row * p.D;
        const float a = lane < p.D ? __ldg(src + lane) : neg_inf();
        const float b = lane + 32 < p.D ? __ldg(src + lane + 32) : neg_inf();
        float m = fmaxf(a, b);
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (!(m > neg_inf())) m = 0.0f;  // impossible step: l = 0
        float* dst = lik + row * 64;
        dst[lane] = ex2((a - m) * kLog2e);
        dst[lane + 32] = ex2((b - m) * kLog2e);
    }
}

// Leaf aggregates of 4 consecutive leaves (2 pairs) per CTA -> p.leafagg (row-major DP x DP, max entry
// in [1,2)); empty leaves get the identity.
__global__ void __launch_bounds__(256, 1) lg_leaf_tc_kernel(const LgParams p, const float* lik) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sBh = smem;           // A^T hi, [n][k] K-major, 16 KB
    uint8_t* sBl = smem + 16384;   // A^T lo
    __shared__ __align__(8) uint64_t mbar[2];
    __shared__ uint32_t tbase;
    __shared__ int emax_s[8];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int pr = warp >> 2, q = warp & 3;
    const int rr = q * 32 + lane;  // row of the stacked operand (= TMEM lane)
    const int h = rr >> 6, r = rr & 63;
    const int64_t T = p.T, SL = p.SL;
    const int64_t nleaves = p.B * p.NL;
    auto leaf_len = [&](int64_t gl) -> int {
        if (gl >= nleaves) return 0;
        const int64_t a = (gl % p.NL) * SL;
        return a < T ? (int)((T - a < SL) ? T - a : SL) : 0;
    };
    const int64_t gl = (int64_t)blockIdx.x * 4 + pr * 2 + h;
    const int64_t gl0 = (int64_t)blockIdx.x * 4 + pr * 2;
    const int n = leaf_len(gl);
    const int nmax = max(leaf_len(gl0), leaf_len(gl0 + 1));
    const int64_t b = gl / p.NL, t0 = (gl % p.NL) * SL;
    uint8_t* Ah = smem + 32768 + (size_t)pr * 65536;
    uint8_t* Al = Ah + 32768;
    const int D = p.D;

    // right operand: B[n][k] = A(k, n), split hi / lo
    for (int i = tid; i < 64 * 64; i += 256) {
        const int nn = i >> 6, k = i & 63;
        const float a = (k < D && nn < D) ? ex2(__ldg(p.log_A + k * D + nn) * kLog2e) : 0.0f;
        const float hi = __uint_as_float(__float_as_uint(a) & 0xffffe000u);
        *reinterpret_cast<float*>(sBh + tc_off(nn, k)) = hi;
        *reinterpret_cast<float*>(sBl + tc_off(nn, k)) = a - hi;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        fence_mbar_init();
    }

    // step 0 of the leaf: row r of psi_{t0} (A(r,:) o l, or pi o l at the sequence's first step)
    int e = 0;
    float v[64];
    if (n > 0) {
        const float4* lr = reinterpret_cast<const float4*>(lik + ((size_t)b * T + t0) * 64);
        const bool first = (p.t_base + t0 == 0);
#pragma unroll
        for (int j4 = 0; j4 < 16; j4++) {
            const float4 l4 = __ldg(lr + j4);
            const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const int j = 4 * j4 + c;
                float a = 0.0f;
                if (j < D && (first || r < D)) a = ex2(__ldg(first ? p.log_pi + j : p.log_A + r * D + j) * kLog2e);
                v[j] = a * lv[c];
            }
        }
        e += row_pow2(v);
        store_split(Ah, Al, rr, v);
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tacc = tbase + (uint32_t)(pr * 64) + ((uint32_t)(q * 32) << 16);
    const uint32_t dcol = tbase + (uint32_t)(pr * 64);

    for (int i = 1; i < nmax; i++) {
        if (q == 0 && lane == 0) {
            tc_fence_after();
            const uint32_t ah = smem_u32(Ah), al = smem_u32(Al), bh = smem_u32(sBh), bl = smem_u32(sBl);
#pragma unroll
            for (int k = 0; k < 8; k++) {
                tc_mma(dcol, tc_desc(ah + 256 * k), tc_desc(bh + 256 * k), k > 0);
                tc_mma(dcol, tc_desc(ah + 256 * k), tc_desc(bl + 256 * k), 1);
                tc_mma(dcol, tc_desc(al + 256 * k), tc_desc(bh + 256 * k), 1);
            }
            tc_commit(&mbar[pr]);
        }
        // the next step's likelihood row, loaded while the MMAs run
        float l[64];
        const bool act = i < n;
        if (act) {
            const float4* lr = reinterpret_cast<const float4*>(lik + ((size_t)b * T + t0 + i) * 64);
#pragma unroll
            for (int j4 = 0; j4 < 16; j4++) {
                const float4 l4 = __ldg(lr + j4);
                l[4 * j4] = l4.x; l[4 * j4 + 1] = l4.y; l[4 * j4 + 2] = l4.z; l[4 * j4 + 3] = l4.w;
            }
        }
        mbar_wait(&mbar[pr], (uint32_t)((i - 1) & 1));
        tc_fence_after();
        tmem_ld64(tacc, v);
        if (act) {
#pragma unroll
            for (int j = 0; j < 64; j++) v[j] *= l[j];
            e += row_pow2(v);
            store_split(Ah, Al, rr, v);
        }
        fence_proxy_async_smem();
        tc_fence_before();
        named_bar(1 + pr, 128);
    }

    // final rows (the operand buffers hold the last stored row of every leaf: hi + lo is exact)
#pragma unroll
    for (int k4 = 0; k4 < 64; k4 += 4) {
        const uint32_t o = tc_off(rr, k4);
        const float4 hh = *reinterpret_cast<const float4*>(Ah + o);
        const float4 ll = *reinterpret_cast<const float4*>(Al + o);
        v[k4] = hh.x + ll.x; v[k4 + 1] = hh.y + ll.y; v[k4 + 2] = hh.z + ll.z; v[k4 + 3] = hh.w + ll.w;
    }
    // fold the row exponents back: scale row r by 2^(e_r - e_max) over the leaf's nonzero rows
    float rs = 0.0f, rmax = 0.0f;
#pragma unroll
    for (int j = 0; j < 64; j++) {
        rs += v[j];
        rmax = fmaxf(rmax, v[j]);
    }
    int eff = (n > 0 && rmax > 0.0f) ? e : INT32_MIN;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) eff = max(eff, __shfl_xor_sync(0xffffffffu, eff, o));
    if (lane == 0) emax_s[warp] = eff;
    __syncthreads();
    const int emax = max(emax_s[warp], emax_s[warp ^ 1]);  // the leaf's two warps
    if (n > 0) {
        const int dd = e - emax;
        const float f = (rmax > 0.0f && dd >= -126) ? __uint_as_float((uint32_t)(dd + 127) << 23) : 0.0f;
        float* dst = p.leafagg + (size_t)gl * 64 * 64 + (size_t)r * 64;
#pragma unroll
        for (int j4 = 0; j4 < 64; j4 += 4)
            *reinterpret_cast<float4*>(dst + j4) = make_float4(v[j4] * f, v[j4 + 1] * f, v[j4 + 2] * f, v[j4 + 3] * f);
        if (rs != rs) atomicOr(reinterpret_cast<uint32_t*>(p.ws_sync + b * 64) + 8, 1u);
    } else if (gl < nleaves) {
        float* dst = p.leafagg + (size_t)gl * 64 * 64 + (size_t)r * 64;
#pragma unroll
        for (int j = 0; j < 64; j++) dst[j] = (j == r) ? 1.0f : 0.0f;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tbase));
}

cudaError_t launch_large_tc_leaf(const LgParams& p, float* lik, cudaStream_t s) {
    const int64_t rows = p.B * p.T;
    const unsigned g1 = (unsigned)((rows + 7) / 8 < 148 * 16 ? (rows + 7) / 8 : 148 * 16);
    lg_lik_kernel<<<g1, 256, 0, s>>>(p, lik);
    const size_t smem = 32768 + 2 * 65536;
    if (cudaError_t e = ensure_smem_optin(reinterpret_cast<const void*>(lg_leaf_tc_kernel), smem); e != cudaSuccess)
        return e;
    const int64_t nleaves = p.B * p.NL;
    lg_leaf_tc_kernel<<<(unsigned)((nleaves + 3) / 4), 256, smem, s>>>(p, lik);
    return cudaGetLastError();
}

}  // namespace hmm
