// hmm_device.cuh — sm_100a device helpers for libhmmscan: TMA bulk copies + mbarrier, grid
// barriers over a sequence's CTAs, pow2 renormalisation, fast exp2, 3-input max.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hmm {

// Host side (hmm_abi.cu): raise `func`'s dynamic shared-memory limit to at least `smem` bytes on the
// CURRENT device.  The attribute is per device, so the record of what was set is keyed by (device,
// kernel) and guarded by a mutex: safe for concurrent first calls and for several GPUs in one process.
cudaError_t ensure_smem_optin(const void* func, size_t smem);

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ float neg_inf() { return __int_as_float(0xff800000); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier + bulk (TMA) copies
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
// Global -> shared bulk copy (cp.async.bulk, SASS UBLKCP), completion counted on `bar`.
// dst/src 16-B aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// Shared -> global bulk copy (bulk_group completion).
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// Per-thread asynchronous global -> shared copies (cp.async, SASS LDGSTS): a normal per-thread
// instruction, unlike UBLKCP whose operands live in uniform registers (per-lane addresses serialise).
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
// zero-filling variant: copies src_bytes (0..16) and fills the rest of the 16 B with zeros
__device__ __forceinline__ void cp_async16_zfill(void* sdst, const void* gsrc, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async8_zfill(void* sdst, const void* gsrc, uint32_t src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async4_zfill(void* sdst, const void* gsrc, uint32_t src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async4(void* sdst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// Make generic-proxy shared-memory writes visible to the async proxy (before a bulk store reads them).
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- global memory ordering
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Longest legitimate wait at a grid barrier is a few milliseconds (the slowest CTA's pass); a wait
// beyond this bound means the counter can never reach G (a workspace left dirty by an aborted launch,
// or CTAs that are not co-resident) and the kernel traps instead of hanging the device.
constexpr unsigned long long kBarrierTimeoutNs = 4000000000ull;  // 4 s

// Arrive-and-wait among the G CTAs of a sequence: every CTA adds 1 (release) and thread 0 spins
// (acquire) until the counter reaches G.  The counters are reset to 0 by the last CTA of the launch
// (after every CTA has passed every wait), so a zero-filled workspace stays valid across calls.
// All G CTAs must be co-resident (cooperative launch).  The spin is bounded (kBarrierTimeoutNs):
// on timeout the launch traps (cudaErrorLaunchFailure on the stream, sticky for the context; the
// caller must then re-zero the workspace, hmmscan.h "Errors").
__device__ __forceinline__ void group_arrive_wait(unsigned long long* counter, uint32_t G) {
    __syncthreads();
    if (threadIdx.x == 0 && G > 1) {
        __threadfence();
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(counter) : "memory");
        if (ld_acquire_u64(counter) < (unsigned long long)G) {
            const unsigned long long t0 = global_ns();
            uint32_t spins = 0;
            while (ld_acquire_u64(counter) < (unsigned long long)G) {
                if ((++spins & 1023u) == 0u && global_ns() - t0 > kBarrierTimeoutNs) __trap();
            }
        }
    }
    __syncthreads();
}

// Copy the G published CTA-root slots (contiguous, slot_bytes a multiple of 16) into the SMEM stage that
// mirrors them: one round of coalesced 16-B L2 loads per thread.  Every CTA of the grid reads the same few
// KB right after the barrier; per-slot scalar loads (16 requests per slot) hot-spotted the few L2 slices
// holding them (3.3 us at G = 148, tools/phase_timers.py).
__device__ __forceinline__ void copy_root_slots(float* stage, const uint8_t* slots, int G, size_t slot_bytes,
                                                int tid, int NT) {
    const int n4 = (int)((size_t)G * slot_bytes / 16);
    const float4* src4 = reinterpret_cast<const float4*>(slots);
    float4* dst4 = reinterpret_cast<float4*>(stage);
    float4 v[4];
#pragma unroll
    for (int j = 0; j < 4; j++)
        if (tid + j * NT < n4) v[j] = __ldcg(src4 + tid + j * NT);
#pragma unroll
    for (int j = 0; j < 4; j++)
        if (tid + j * NT < n4) dst4[tid + j * NT] = v[j];
    for (int i = tid + 4 * NT; i < n4; i += NT) dst4[i] = __ldcg(src4 + i);
}

// ---------------------------------------------------------------- arithmetic helpers
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float max3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
// Exponent offset d = 127 - E(m) (E = biased exponent), as an exact float: m * 2^d lies in [1,2) for a
// positive normal m.  Used as an additive term of an ex2 argument, so applying the power-of-two
// renormalisation costs no multiplies.  Built with the 2^23 magic constant (no I2F).
__device__ __forceinline__ float exp_offset(float m) {
    const float biased = __uint_as_float((__float_as_uint(m) >> 23) | 0x4B000000u);  // 2^23 + E (m >= 0)
    return 8388735.0f - biased;                                                      // (2^23 + 127) - (2^23 + E)
}
// Max of N values with 2-input FMNMX (full rate on sm_100; the 3-input FMNMX3 issues at half rate,
// tools/microbench/pipes.cu) as a balanced tree.
template <int N>
__device__ __forceinline__ float vmax2_tree(const float* v) {
    if constexpr (N == 1) {
        return v[0];
    } else {
        constexpr int H = N / 2;
        return fmaxf(vmax2_tree<H>(v), vmax2_tree<N - H>(v + H));
    }
}
// Max of N values by a 3-ary tree (depth ~log3 N instead of a serial chain).
template <int N>
__device__ __forceinline__ float vmax_tree(const float* v) {
    if constexpr (N <= 3) {
        if constexpr (N == 1) return v[0];
        else if constexpr (N == 2) return fmaxf(v[0], v[1]);
        else return max3(v[0], v[1], v[2]);
    } else {
        constexpr int G = (N + 2) / 3;
        float w[G];
#pragma unroll
        for (int g = 0; g < G; g++) {
            const int a = 3 * g;
            if (a + 2 < N) w[g] = max3(v[a], v[a + 1], v[a + 2]);
            else if (a + 1 < N) w[g] = fmaxf(v[a], v[a + 1]);
            else w[g] = v[a];
        }
        return vmax_tree<G>(w);
    }
}
// Exact power-of-two factor s with m*s in [1,2) for a positive normal m; 1 for 0 / denormal / huge.
__device__ __forceinline__ float pow2_inv(float m) {
    uint32_t e = __float_as_uint(m) & 0x7f800000u;
    uint32_t s = 0x7f000000u - e;  // biased exponent 254 - e
    return (e == 0u || e >= 0x7f000000u) ? 1.0f : __uint_as_float(s);
}
template <int N>
__device__ __forceinline__ float vmax(const float* v) {
    if constexpr (N == 1) {
        return v[0];
    } else if constexpr (N == 2) {
        return fmaxf(v[0], v[1]);
    } else {
        float m = max3(v[0], v[1], v[2]);
        int i = 3;
#pragma unroll
        for (; i + 1 < N; i += 2) m = max3(m, v[i], v[i + 1]);
        if (i < N) m = fmaxf(m, v[i]);
        return m;
    }
}
template <int N>
__device__ __forceinline__ float vsum(const float* v) {
    float s = v[0];
#pragma unroll
    for (int i = 1; i < N; i++) s += v[i];
    return s;
}

}  // namespace hmm
