// hmm_batchseq.cu — batch-parallel plan for many sequences with 9 <= D <= 32 (SURVEY.md §8(a) a9,
// BASELINE config ④: B = 1024, D = 16, T = 4096), sm_100a.
//
// With B sequences the batch alone fills the GPU, so the scan's per-step D x D element products
// (D^3 work) are pure overhead: each sequence is one block-wise element spanning the whole sequence
// ("a single computational element to a set of consecutive observations"), evaluated
// by the element recursions themselves — Algorithm 1's forward and backward passes (PAPER.md:156-174,
// D^2 work per step) and Algorithm 4's forward max-product pass with backpointers.
// The planner picks this plan when B is large enough that the scan's D^3 work costs more than the
// recursions' latency (hmm_abi.cu); the scan plans stay for small B.
//
// One group of DP lanes (DP = 16: half a warp, DP = 32: a warp) owns a sequence; lane j holds state j.
// A step gathers the previous vector with DP shuffles, so every lane also sees the whole vector: the
// exact power-of-two renormalisation (sum-product) or the max subtraction (max-product) is computed
// redundantly from the gathered values — no reduction on the recursion's critical path — and the
// normalised outputs of step t are produced one step later, off it.  The vector exchange goes through a
// per-group SMEM slot (one store, __syncwarp, broadcast LDS.128 reads) and the log_lik / filtered rows
// are staged in SMEM chunks of kBsC steps by cp.async, two chunks ahead of the one in use (the
// per-step loads of a register prefetch did not cover the memory latency at this step rate).
//
//   bs_smooth   forward: a_t = s_t ((a_{t-1} A) o l_t), s_t = 2^k from max(a_{t-1}); filtered_{t-1}
//               = a_{t-1}/sum; log Z = log sum(a_{T-1}) - sum log s_t + sum m_t (exact telescoping).
//               backward: b_{t-1} = s (A (l_t o b_t)); smoothed_t = f_t o b_t / sum (Eq. 14), f_t the
//               filtered row read back.
//   bs_viterbi  forward: V~_t(j) = max_i (V~_{t-1}(i) - o_{t-1} + log A(i,j)) + w_t(j), backpointer =
//               smallest maximising i (one byte per state per step, workspace); then the backtrack,
//               staged through shared memory in chunks.
#include <cfloat>
#include <cstdint>
#include <cstring>

#include "hmm_device.cuh"
#include "hmm_large.h"
#include "hmm_plan.h"

namespace hmm {


constexpr int kBsThreads = 128;
constexpr int kBsC = 32;      // steps per staged chunk
constexpr int kBsStages = 3;  // chunk ring depth (two chunks in flight ahead of the one in use)
constexpr int kBsChunk = 256;  // backtrack chunk (steps)

template <int DP>
__device__ __forceinline__ unsigned bs_mask() {
    if constexpr (DP == 32) return 0xffffffffu;
    else return 0xffffu << (16 * ((threadIdx.x >> 4) & 1));
}
// log2 of the exact power-of-two factor pow2_inv(m) (0 when pow2_inv returns 1)
__device__ __forceinline__ int pow2_inv_log2(float m) {
    const uint32_t e = (__float_as_uint(m) >> 23) & 0xffu;
    return (e == 0u || e >= 0xfeu) ? 0 : 127 - (int)e;
}
// Balanced trees (depth log2 N instead of an N-deep chain: the reductions sit on the recursion's
// critical path, and the compiler may not reassociate fp adds).
template <int N>
__device__ __forceinline__ float tmax(const float* v) {
    if constexpr (N == 1) return v[0];
    else if constexpr (N == 2) return fmaxf(v[0], v[1]);
    else return fmaxf(tmax<N / 2>(v), tmax<N - N / 2>(v + N / 2));
}
template <int N>
__device__ __forceinline__ float tsum(const float* v) {
    if constexpr (N == 1) return v[0];
    else if constexpr (N == 2) return v[0] + v[1];
    else return tsum<N / 2>(v) + tsum<N - N / 2>(v + N / 2);
}
// smallest k with v[k] == best (best = max v): equality bits OR-ed by a tree, then the lowest set bit
template <int N>
__device__ __forceinline__ uint32_t eq_bits(const float* v, float best, int k0) {
    if constexpr (N == 1) return (v[0] == best) ? (1u << k0) : 0u;
    else return eq_bits<N / 2>(v, best, k0) | eq_bits<N - N / 2>(v + N / 2, best, k0 + N / 2);
}
template <int N>
__device__ __forceinline__ int first_argmax(const float* v, float best) {
    const uint32_t m = eq_bits<N>(v, best, 0);
    return m ? __ffs(m) - 1 : 0;
}
template <int N>
__device__ __forceinline__ void ld_vec(const float* p, float* v) {
#pragma unroll
    for (int i = 0; i < N; i += 4) {
        const float4 x = *reinterpret_cast<const float4*>(p + i);
        v[i] = x.x; v[i + 1] = x.y; v[i + 2] = x.z; v[i + 3] = x.w;
    }
}

// One warp per sequence: lane = (state j = lane % DP, half h = lane / DP), H = 32 / DP halves (2 for
// DP = 16: two lanes per state split every dot product and reduction, so the batch of config ④ gives
// twice as many warps to hide the recursion's latency).  NV = DP / H values per lane.
template <int DP> struct BsShape {
    static constexpr int H = 32 / DP;
    static constexpr int NV = DP / H;
};

// Per-sequence staging of rows in SMEM: chunk c = rows [c C, c C + C) of a [T][D] array, row pitch DP
// floats, element (r, j) copied by lane (j, r % H) with 4-B cp.async (any D, any row alignment),
// kBsStages-deep ring, one cp.async group per chunk.
template <int DP>
struct BsRing {
    float* buf;  // [kBsStages][kBsC][DP]
    const float* src;
    int64_t T;
    int D, j, h;
    __device__ __forceinline__ float* stage(int64_t c) const { return buf + (size_t)(c % kBsStages) * kBsC * DP; }
    __device__ __forceinline__ void issue(int64_t c) const {
        if (c >= 0 && c * kBsC < T && j < D) {
            const int64_t r0 = c * kBsC;
            const int n = (int)((T - r0 < kBsC) ? T - r0 : kBsC);
            float* dst = stage(c) + j;
            const float* s = src + r0 * D + j;
            for (int r = h; r < n; r += BsShape<DP>::H) cp_async4(dst + r * DP, s + (int64_t)r * D);
        }
        cp_async_commit();
    }
};

template <int DP>
__device__ __forceinline__ void bs_fill(float* buf, int nfl, float v) {
    for (int e = threadIdx.x % 32; e < nfl; e += 32) buf[e] = v;
}

// Chunk preparation: row r's maximum m_r = max_{j<D} ll_r(j) (lane r, kBsC = 32 rows) and a NaN / +inf
// flag, then every element turned into l = exp(ll - m_r) (sum-product) or w = ll - m_r (max-product);
// padded states get l = 0 / w = -inf.  The per-step recursion then reads one value.
template <int DP, bool MP>
__device__ __forceinline__ bool bs_prep(float* rows, float* mrow, int n, int D, int j, int h) {
    const int lane = threadIdx.x % 32;
    bool bad = false;
    if (lane < n) {
        float v[DP];
        ld_vec<DP>(rows + lane * DP, v);
        float cs = 0.0f;
#pragma unroll
        for (int k = 0; k < DP; k++) {
            cs += (k < D) ? v[k] : 0.0f;
            v[k] = (k < D) ? v[k] : neg_inf();
        }
        const float m = tmax<DP>(v);
        bad = (cs != cs) || (cs == INFINITY);
        mrow[lane] = (m > -FLT_MAX) ? m : 0.0f;  // impossible step: l = 0 / w = -inf, caught downstream
    }
    __syncwarp();
    for (int r = h; r < n; r += BsShape<DP>::H) {
        const float x = rows[r * DP + j] - mrow[r];
        rows[r * DP + j] = (j < D) ? (MP ? x : ex2(x * kLog2e)) : (MP ? neg_inf() : 0.0f);
    }
    __syncwarp();
    return __any_sync(0xffffffffu, bad);
}

// Normalise n staged rows and store them coalesced to dst rows [0, n) (pitch D).  Returns the first
// zero-mass row (or -1) and the sum of row n-1 in `last`.
template <int DP>
__device__ __forceinline__ int bs_flush(float* rows, int n, float* dst, int D, int j, int h, float* inv, bool& bad,
                                        float& last) {
    const int lane = threadIdx.x % 32;
    float sm = 1.0f;
    if (lane < n) {
        float v[DP];
        ld_vec<DP>(rows + lane * DP, v);
        sm = tsum<DP>(v);
        inv[lane] = (sm > 0.0f) ? rcp(sm) : 0.0f;
    }
    const uint32_t zmask = __ballot_sync(0xffffffffu, lane < n && !(sm > 0.0f));
    bad |= __any_sync(0xffffffffu, sm != sm);
    last = __shfl_sync(0xffffffffu, sm, n - 1);
    __syncwarp();
    if (j < D)
        for (int r = h; r < n; r += BsShape<DP>::H) dst[(int64_t)r * D + j] = rows[r * DP + j] * inv[r];
    __syncwarp();
    return zmask ? __ffs(zmask) - 1 : -1;
}

template <int DP>
__global__ void __launch_bounds__(kBsThreads) bs_smooth_kernel(const BSParams p) {
    using S = BsShape<DP>;
    constexpr int H = S::H, NV = S::NV;
    constexpr int SPB = kBsThreads / 32;
    constexpr int RING = kBsStages * kBsC * DP;
    constexpr int OUT = (kBsC + 1) * DP;
    constexpr int PER = 2 * RING + OUT + 2 * kBsC;
    extern __shared__ __align__(16) float bsm[];
    const int lane = threadIdx.x % 32, grp = threadIdx.x / 32;
    const int j = lane % DP, h = lane / DP;
    float* rl_buf = bsm + (size_t)grp * PER;  // log_lik chunks (turned into l in place)
    float* rf_buf = rl_buf + RING;            // filtered chunks (backward pass)
    float* out = rf_buf + RING;               // [1 + C][DP]: row 0 = previous step, rows 1.. = this chunk
    float* mrow = out + OUT;                  // [C] row maxima m_t
    float* inv = mrow + kBsC;                 // [C] row normalisers
    const int64_t b = (int64_t)blockIdx.x * SPB + grp;
    if (b >= p.B) return;
    int64_t base, raw;
    const int64_t T = seq_span(p.offsets, p.T, b, base, raw);
    if (T < 1) {  // (varlen: invalid length)
        if (lane == 0) { p.scalar_out[b] = 0.0; p.info[b] = kInfoBadLength; }
        return;
    }
    const int D = p.D;
    const bool act = j < D;
    const float* la = p.log_A + b * p.A_stride;
    float Acol[NV], Arow[NV];  // A(i, j) and A(j, i) for i in this lane's half
#pragma unroll
    for (int k = 0; k < NV; k++) {
        const int i = h * NV + k;
        Acol[k] = (act && i < D) ? ex2(__ldg(la + i * D + j) * kLog2e) : 0.0f;
        Arow[k] = (act && i < D) ? ex2(__ldg(la + j * D + i) * kLog2e) : 0.0f;
    }
    const float piv = act ? ex2(__ldg(p.log_pi + b * p.pi_stride + j) * kLog2e) : 0.0f;
    float* filt = p.filtered + base * D;
    float* smo = p.smoothed + base * D;
    bs_fill<DP>(rl_buf, 2 * RING + OUT, 0.0f);  // pads of the filtered ring and the staging rows stay 0
    __syncwarp();
    const BsRing<DP> rl{rl_buf, p.log_lik + base * D, T, D, j, h};
    const BsRing<DP> rf{rf_buf, filt, T, D, j, h};
    const int64_t nch = (T + kBsC - 1) / kBsC;
    auto hsum = [&](float v) -> float { return (H == 2) ? v + __shfl_xor_sync(0xffffffffu, v, 16) : v; };
    auto hmax = [&](float v) -> float { return (H == 2) ? fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 16)) : v; };

    // ---------------- forward (Algorithm 1 forward pass): a_t = s_t ((a_{t-1} A) o l_t), staged in `out`
    // (the staged row is also the vector exchange), normalised per chunk into filtered.
    double msum = 0.0;
    int es = 0;           // sum of log2 s_t
    int64_t zero_t = -1;  // first step with zero forward mass
    bool bad = false;
    float lastsum = 0.0f;
    rl.issue(0);
    rl.issue(1);
    for (int64_t c = 0; c < nch; c++) {
        rl.issue(c + 2);
        cp_async_wait<2>();
        __syncwarp();
        float* rows = rl.stage(c);
        const int n = (int)((T - c * kBsC < kBsC) ? T - c * kBsC : kBsC);
        bad |= bs_prep<DP, false>(rows, mrow, n, D, j, h);
        for (int i = 0; i < n; i++) msum += (double)mrow[i];
        for (int i = 0; i < n; i++) {
            const int64_t t = c * kBsC + i;
            const float l = rows[i * DP + j];
            float a;
            if (t == 0) {
                a = piv * l;
            } else {
                float g[NV];
                ld_vec<NV>(out + i * DP + h * NV, g);  // this half of a_{t-1}
                const float mx = hmax(tmax<NV>(g));
                const float s = pow2_inv(mx);
                es += pow2_inv_log2(mx);
                float c0 = 0.0f, c1 = 0.0f, c2 = 0.0f, c3 = 0.0f;
#pragma unroll
                for (int k = 0; k < NV; k += 4) {
                    c0 = fmaf(g[k], Acol[k], c0);
                    c1 = fmaf(g[k + 1], Acol[k + 1], c1);
                    c2 = fmaf(g[k + 2], Acol[k + 2], c2);
                    c3 = fmaf(g[k + 3], Acol[k + 3], c3);
                }
                a = hsum((c0 + c1) + (c2 + c3)) * (l * s);
            }
            if (h == 0) out[(i + 1) * DP + j] = a;
            __syncwarp();
        }
        const int z = bs_flush<DP>(out + DP, n, filt + c * kBsC * D, D, j, h, inv, bad, lastsum);
        if (z >= 0 && zero_t < 0) zero_t = c * kBsC + z;
        if (h == 0) out[j] = out[n * DP + j];  // carry a_{t0-1} into row 0
        __syncwarp();
    }
    const double logz = log((double)lastsum) - (double)es * (double)kLn2 + msum;
    cp_async_wait<0>();
    __syncwarp();  // the filtered rows of the sequence are complete before the backward pass stages them

    // ---------------- backward (Algorithm 1 backward pass) + Eq. 14, chunks in reverse order: the staged
    // l row of step t becomes w = l_t o b_t (the exchange for b_{t-1}); gam_t = f_t o b_t is staged in
    // `out` and normalised per chunk into smoothed.
    float bt = act ? 1.0f : 0.0f;  // b_{T-1} = 1 (Thm 2: a_{T:T+1} = 1)
    rl.issue(nch - 1); rf.issue(nch - 1);
    rl.issue(nch - 2); rf.issue(nch - 2);
    for (int64_t c = nch - 1; c >= 0; c--) {
        rl.issue(c - 2); rf.issue(c - 2);
        cp_async_wait<4>();
        __syncwarp();
        float* rows = rl.stage(c);
        const float* frows = rf.stage(c);
        const int n = (int)((T - c * kBsC < kBsC) ? T - c * kBsC : kBsC);
        bs_prep<DP, false>(rows, mrow, n, D, j, h);
        for (int i = n - 1; i >= 0; i--) {
            const int64_t t = c * kBsC + i;
            if (h == 0) {
                out[(i + 1) * DP + j] = frows[i * DP + j] * bt;  // gam_t (unnormalised)
                rows[i * DP + j] *= bt;                           // w = l_t o b_t (pads: 0)
            }
            __syncwarp();
            if (t > 0) {  // b_{t-1} = A (l_t o b_t), renormalised by an exact power of two
                float g[NV];
                ld_vec<NV>(rows + i * DP + h * NV, g);
                const float s = pow2_inv(hmax(tmax<NV>(g)));
                float c0 = 0.0f, c1 = 0.0f, c2 = 0.0f, c3 = 0.0f;
#pragma unroll
                for (int k = 0; k < NV; k += 4) {
                    c0 = fmaf(Arow[k], g[k], c0);
                    c1 = fmaf(Arow[k + 1], g[k + 1], c1);
                    c2 = fmaf(Arow[k + 2], g[k + 2], c2);
                    c3 = fmaf(Arow[k + 3], g[k + 3], c3);
                }
                bt = hsum((c0 + c1) + (c2 + c3)) * s;
            }
        }
        __syncwarp();
        bool dummy = false;
        float dl;
        bs_flush<DP>(out + DP, n, smo + c * kBsC * D, D, j, h, inv, dummy, dl);
    }
    cp_async_wait<0>();
    if (lane == 0) {
        p.scalar_out[b] = logz;
        int32_t inf = 0;
        if (bad || logz != logz) inf = -1;
        else if (zero_t >= 0) inf = (int32_t)(zero_t + 1);
        if (raw < 1 || raw > p.T) inf = kInfoBadLength;
        p.info[b] = inf;
    }
}

template <int DP>
__global__ void __launch_bounds__(kBsThreads) bs_viterbi_kernel(const BSParams p) {
    using S = BsShape<DP>;
    constexpr int H = S::H, NV = S::NV;
    constexpr int SPB = kBsThreads / 32;
    constexpr int RING = kBsStages * kBsC * DP;
    constexpr int PER = RING + 2 * DP + kBsC + kBsChunk + kBsChunk * DP / 4;
    extern __shared__ __align__(16) float bsm[];
    const int lane = threadIdx.x % 32, grp = threadIdx.x / 32;
    const int j = lane % DP, h = lane / DP;
    float* rl_buf = bsm + (size_t)grp * PER;
    float* xbuf = rl_buf + RING;                                     // [2][DP]
    float* mrow = xbuf + 2 * DP;                                     // [C]
    int32_t* spath = reinterpret_cast<int32_t*>(mrow + kBsC);        // [kBsChunk]
    uint8_t* sbp = reinterpret_cast<uint8_t*>(spath + kBsChunk);     // [kBsChunk][DP]
    const int64_t b = (int64_t)blockIdx.x * SPB + grp;
    if (b >= p.B) return;
    int64_t base, raw;
    const int64_t T = seq_span(p.offsets, p.T, b, base, raw);
    if (T < 1) {
        if (lane == 0) { p.scalar_out[b] = 0.0; p.info[b] = kInfoBadLength; }
        return;
    }
    const int D = p.D;
    const bool act = j < D;
    const float* la = p.log_A + b * p.A_stride;
    float LA[NV];  // log A(i, j) for i in this lane's half
#pragma unroll
    for (int k = 0; k < NV; k++) {
        const int i = h * NV + k;
        LA[k] = (act && i < D) ? __ldg(la + i * D + j) : neg_inf();
    }
    const float lpv = act ? __ldg(p.log_pi + b * p.pi_stride + j) : neg_inf();
    uint8_t* bp = p.bp + (size_t)b * p.T * DP;
    bs_fill<DP>(rl_buf, RING + 2 * DP, neg_inf());
    __syncwarp();
    const BsRing<DP> rl{rl_buf, p.log_lik + base * D, T, D, j, h};
    const int64_t nch = (T + kBsC - 1) / kBsC;

    // ---------------- forward max-product pass with backpointers (Algorithm 4 lines 3-6)
    double c = 0.0;  // accumulated offset: V_t = V~_t + c
    int64_t zero_t = -1;
    bool bad = false;
    float V = neg_inf();
    int par = 0;
    rl.issue(0);
    rl.issue(1);
    for (int64_t ch = 0; ch < nch; ch++) {
        rl.issue(ch + 2);
        cp_async_wait<2>();
        __syncwarp();
        float* rows = rl.stage(ch);
        const int n = (int)((T - ch * kBsC < kBsC) ? T - ch * kBsC : kBsC);
        bad |= bs_prep<DP, true>(rows, mrow, n, D, j, h);
        for (int i = 0; i < n; i++) {
            const int64_t t = ch * kBsC + i;
            const float w = rows[i * DP + j];
            const float m = mrow[i];
            if (t == 0) {
                V = lpv + w;
                c = (double)m;
            } else {
                float* xb = xbuf + par * DP;
                par ^= 1;
                if (h == 0) xb[j] = V;
                __syncwarp();
                float g[NV];
                ld_vec<NV>(xb + h * NV, g);
                float o = tmax<NV>(g);
                if (H == 2) o = fmaxf(o, __shfl_xor_sync(0xffffffffu, o, 16));
                if (!(o > neg_inf())) {
                    if (zero_t < 0) zero_t = t - 1;
                    o = 0.0f;
                }
                float sc[NV];
#pragma unroll
                for (int k = 0; k < NV; k++) sc[k] = (g[k] - o) + LA[k];
                float best = tmax<NV>(sc);
                int arg = first_argmax<NV>(sc, best) + h * NV;
                if (H == 2) {  // the lower half wins ties (smallest index)
                    const float bo = __shfl_xor_sync(0xffffffffu, best, 16);
                    const int ao = __shfl_xor_sync(0xffffffffu, arg, 16);
                    const float bl = h ? bo : best, bh = h ? best : bo;
                    const int al = h ? ao : arg, ah = h ? arg : ao;
                    best = fmaxf(bl, bh);
                    arg = (bl == best) ? al : ah;
                }
                if (h == 0 && act) bp[t * DP + j] = (uint8_t)arg;
                V = best + w;
                c += (double)o + (double)m;
            }
        }
        __syncwarp();
    }
    cp_async_wait<0>();
    // x*_{T-1} = smallest argmax of V_{T-1}; log_prob = max V_{T-1}
    int xs;
    {
        float* xb = xbuf + par * DP;
        if (h == 0) xb[j] = V;
        __syncwarp();
        float g[DP];
        ld_vec<DP>(xb, g);
        float o = tmax<DP>(g);
        xs = first_argmax<DP>(g, o);
        if (!(o > neg_inf())) {
            if (zero_t < 0) zero_t = T - 1;
            o = 0.0f;
            xs = 0;
        }
        c += (double)o;
    }
    __syncwarp();  // the backpointer stores are visible to all lanes
    // ---------------- backtrack (Algorithm 4 lines 8-10), chunks of the backpointers staged in SMEM
    int x = xs;
    for (int64_t e = T; e > 0; e -= kBsChunk) {
        const int64_t s0 = (e - kBsChunk > 0) ? e - kBsChunk : 0;
        const int n = (int)(e - s0);
        const uint32_t* src = reinterpret_cast<const uint32_t*>(bp + s0 * DP);
        uint32_t* dst = reinterpret_cast<uint32_t*>(sbp);
        for (int q = lane; q < n * DP / 4; q += 32) dst[q] = src[q];
        __syncwarp();
        if (lane == 0) {
            for (int i = n - 1; i >= 0; i--) {
                spath[i] = x;
                if (s0 + i > 0) x = sbp[i * DP + x];
            }
        }
        __syncwarp();
        for (int i = lane; i < n; i += 32) p.path[base + s0 + i] = spath[i];
        __syncwarp();
    }
    if (lane == 0) {
        p.scalar_out[b] = c;
        int32_t inf = 0;
        if (bad || c != c) inf = -1;
        else if (zero_t >= 0) inf = (int32_t)(zero_t + 1);
        if (raw < 1 || raw > p.T) inf = kInfoBadLength;
        p.info[b] = inf;
    }
}

// ============================================================================ bidirectional plan
// Two recursions per sequence running at the same time from the two ends and meeting in the middle: the
// forward recursion (Algorithm 1 forward / Algorithm 4 forward) and the backward recursion (Algorithm 1
// backward / the max-product backward recursion of Lemma 3), so a sequence takes T
// recursion steps of latency instead of 2T (sum-product) or T + the backtrack (max-product).  The
// sequence is cut at mid = ceil(nch / 2) chunks:
//   smoother  phase 1: forward over [0, mid) (filtered) | backward over [mid, T) (b_t kept in the
//             workspace);  phase 2: forward over [mid, T) (filtered, smoothed = a_t o b_t / sum from the
//             kept b_t) | backward over [0, mid) (smoothed from the filtered rows of phase 1).
//   Viterbi   forward max-product over [0, mid) with backpointers | backward max-product over [mid, T)
//             with forward pointers; x*_{mid-1} = argmax (V^f + V^b) (Theorem 4's max-marginal at one
//             step, smallest index), log_prob = its value; then both halves of the path in parallel
//             (backtrack / forward track).
// Layout: a CTA = 2 warps (warp 0 forward, warp 1 backward) x G = 32 / DP sequences per warp; lane group
// g (DP lanes) of a warp serves sequence 2 b0 + g, lane j of a group holds state j and computes its whole
// dot product (no half-warp split: at DP = 16 two sequences share each warp instruction, the plan is
// issue-bound at config 4's batch).  One CTA barrier separates the phases; everything else is per lane
// group (group masks: sequences of one warp may differ in length).  Chunk rings are 2 deep (a chunk is
// ~6 us of recursion, far above the load latency).
constexpr int kBs2Threads = 64;
constexpr int kBs2Stages = 2;

template <int DP> struct Bs2 {
    static constexpr int G = 32 / DP;                        // sequences per warp
    static constexpr int RING = kBs2Stages * kBsC * DP;      // floats per chunk ring
    static constexpr int VT_PER = RING + 2 * DP + kBsC + kBsChunk + kBsChunk * DP / 4;  // Viterbi
};
template <int DP>
__device__ __forceinline__ unsigned bs2_gmask(int g) {
    if constexpr (DP == 32) return 0xffffffffu;
    else return 0xffffu << (16 * g);
}
// Visit the (row, quad) pairs of n rows x nq 16-B quads with lane j taking pairs j, j + DP, ..; when nq
// divides DP the pair index splits without a division (q = j % nq fixed, r advances by DP / nq).
template <int DP, int NQ, class F>
__device__ __forceinline__ void for_quads_c(int n, int j, F&& f) {
    constexpr int RS = DP / NQ;  // (NQ divides DP: q fixed per lane, rows advance by DP / NQ)
    const int q = j % NQ;
    for (int r = j / NQ; r < n; r += RS) f(r, q);
}
template <int DP, class F>
__device__ __forceinline__ void for_quads(int n, int nq, int j, F&& f) {
    switch (nq) {  // compile-time divisors of DP: shifts instead of integer divisions
        case 1: for_quads_c<DP, 1>(n, j, f); return;
        case 2: for_quads_c<DP, 2>(n, j, f); return;
        case 4: for_quads_c<DP, 4>(n, j, f); return;
        case 8: if constexpr (DP % 8 == 0) { for_quads_c<DP, 8>(n, j, f); return; } break;
        default: break;
    }
    for (int e = j; e < n * nq; e += DP) {
        const int r = e / nq;
        f(r, e - r * nq);
    }
}
// per-group staging ring: element (r, j) of chunk c copied by lane j (4-B cp.async, any D / alignment)
template <int DP>
struct Bs2Ring {
    float* buf;  // [kBs2Stages][kBsC][DP]
    const float* src;
    int64_t T;
    int D, j;
    __device__ __forceinline__ float* stage(int64_t c) const { return buf + (size_t)((uint32_t)c % (uint32_t)kBs2Stages) * kBsC * DP; }
    bool vec;    // D % 4 == 0 and 16-B aligned rows: 16-B copies
    __device__ __forceinline__ void issue(int64_t c, bool live) const {
        if (live && c >= 0 && c * kBsC < T) {
            const int64_t r0 = c * kBsC;
            const int n = (int)((T - r0 < kBsC) ? T - r0 : kBsC);
            if (vec) {
                float* dst = stage(c);
                const float* s = src + r0 * D;
                const int Dl = D;
                for_quads<DP>(n, D >> 2, j, [&](int r, int q) { cp_async16(dst + r * DP + 4 * q, s + (int64_t)r * Dl + 4 * q); });
            } else if (j < D) {
                float* dst = stage(c) + j;
                const float* s = src + r0 * D + j;
                for (int r = 0; r < n; r++) cp_async4(dst + r * DP, s + (int64_t)r * D);
            }
        }
        cp_async_commit();
    }
};
__device__ __forceinline__ bool bs2_vec_ok(const void* p, int D) {
    return (D & 3) == 0 && (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}
// chunk preparation per group (as bs_prep): row maxima m_r (lane j handles rows j, j + DP, ..), NaN / +inf
// flag, then l = exp(ll - m) / w = ll - m in place (pads: 0 / -inf)
template <int DP, bool MP>
__device__ __forceinline__ bool bs2_prep(float* rows, float* mrow, int n, int D, int j, unsigned gm,
                                         double* msum = nullptr) {
    bool bad = false;
    for (int r = j; r < n; r += DP) {
        float v[DP];
        ld_vec<DP>(rows + r * DP, v);
        float cs = 0.0f;
#pragma unroll
        for (int k = 0; k < DP; k++) {
            if constexpr (MP) cs += (k < D) ? v[k] : 0.0f;
            v[k] = (k < D) ? v[k] : neg_inf();
        }
        const float m = tmax<DP>(v);
        // max-plus: FMNMX drops NaN, so NaN / +inf inputs are flagged here; sum-product: they reach the
        // forward rows (l = exp(NaN)) and the filtered flush's row sums flag them
        if constexpr (MP) bad |= (cs != cs) || (cs == INFINITY);
        mrow[r] = (m > -FLT_MAX) ? m : 0.0f;
        if (msum) *msum += (double)mrow[r];  // this lane's share of sum m_t (rows j, j + DP, ..)
    }
    __syncwarp(gm);
    constexpr int QP = DP / 4;  // quads per staged row (pads included)
    for (int e = j; e < n * QP; e += DP) {
        const int r = e / QP, q = e - r * QP;
        float4* pr = reinterpret_cast<float4*>(rows + r * DP) + q;
        const float4 x4 = *pr;
        const float m = mrow[r];
        float x[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const float d = x[u] - m;
            x[u] = (4 * q + u < D) ? (MP ? d : ex2(d * kLog2e)) : (MP ? neg_inf() : 0.0f);
        }
        *pr = make_float4(x[0], x[1], x[2], x[3]);
    }
    __syncwarp(gm);
    return bad;  // lane-local: callers OR it over the lane group once, at the end
}
// normalise n staged rows and store them to dst (pitch D); first zero-mass row (or -1), sum of row n-1
template <int DP, bool ZERO = true>
__device__ __forceinline__ int bs2_flush(const float* rows, int n, float* dst, int D, int j, unsigned gm, float* inv,
                                         bool& bad, float& last, bool vec) {
    uint32_t zm = 0u;
    bool nan = false;
    float mylast = 0.0f;
    for (int r = j; r < n; r += DP) {
        float v[DP];
        ld_vec<DP>(rows + r * DP, v);
        const float sm = tsum<DP>(v);
        inv[r] = (sm > 0.0f) ? rcp(sm) : 0.0f;
        if (!(sm > 0.0f)) zm |= 1u << r;
        nan |= (sm != sm);
        if (r == n - 1) mylast = sm;
    }
    __syncwarp(gm);
    // OR of the groups' zero masks (bit r = row r), first set bit
    if constexpr (ZERO) {
#pragma unroll
        for (int o = DP / 2; o >= 1; o >>= 1) zm |= __shfl_xor_sync(gm, zm, o, DP);
    }
    bad |= nan;  // lane-local (OR-ed over the lane group at the end)
    last = __shfl_sync(gm, mylast, (n - 1) % DP, DP);  // the row sum of row n-1, from the lane that took it
    if (vec) {  // 16-B stores: lane j takes quads j, j + DP, .. of the chunk's n x D/4
        for_quads<DP>(n, D >> 2, j, [&](int r, int q) {
            const float4 v = reinterpret_cast<const float4*>(rows + r * DP)[q];
            const float iv = inv[r];
            reinterpret_cast<float4*>(dst + (int64_t)r * D)[q] = make_float4(v.x * iv, v.y * iv, v.z * iv, v.w * iv);
        });
    } else if (j < D) {
        for (int r = 0; r < n; r++) dst[(int64_t)r * D + j] = rows[r * DP + j] * inv[r];
    }
    __syncwarp(gm);
    return zm ? __ffs(zm) - 1 : -1;
}

template <int DP>
__global__ void __launch_bounds__(kBs2Threads) bs2_viterbi_kernel(const BSParams p) {
    using Z = Bs2<DP>;
    constexpr int G = Z::G, RING = Z::RING, PER = Z::VT_PER;
    extern __shared__ __align__(16) float bsm[];
    __shared__ float vmeet[G][2][DP];
    __shared__ double cmeet[G];
    __shared__ int fmeet[G];
    const int lane = threadIdx.x % 32, role = threadIdx.x / 32;  // role 0: forward, 1: backward
    const int g = lane / DP, j = lane % DP;
    const unsigned gm = bs2_gmask<DP>(g);
    float* rl_buf = bsm + (size_t)(role * G + g) * PER;
    float* xbuf = rl_buf + RING;                                  // [2][DP]
    float* mrow = xbuf + 2 * DP;                                  // [C]
    int32_t* spath = reinterpret_cast<int32_t*>(mrow + kBsC);     // [kBsChunk]
    uint8_t* sbp = reinterpret_cast<uint8_t*>(spath + kBsChunk);  // [kBsChunk][DP]
    const int64_t b = (int64_t)blockIdx.x * G + g;
    int64_t base = 0, raw = 0, T = 0;
    if (b < p.B) T = seq_span(p.offsets, p.T, b, base, raw);
    const bool live = T >= 1;
    if (b < p.B && !live && role == 0 && j == 0) { p.scalar_out[b] = 0.0; p.info[b] = kInfoBadLength; }
    const int D = p.D;
    const bool act = j < D;
    const float* la = p.log_A + (b < p.B ? b : 0) * p.A_stride;
    float LA[DP];  // forward: log A(i, j); backward: log A(j, i)
#pragma unroll
    for (int i = 0; i < DP; i++)
        LA[i] = (act && i < D && live) ? __ldg(role == 0 ? la + i * D + j : la + j * D + i) : neg_inf();
    const float lpv = (act && live) ? __ldg(p.log_pi + b * p.pi_stride + j) : neg_inf();
    uint8_t* bp = p.bp + (size_t)(b < p.B ? b : 0) * p.T * DP;
    for (int e = j; e < RING + 2 * DP; e += DP) rl_buf[e] = neg_inf();
    __syncwarp(gm);
    const Bs2Ring<DP> rl{rl_buf, p.log_lik + base * D, T, D, j, bs2_vec_ok(p.log_lik, D)};
    const int64_t nch = (T + kBsC - 1) / kBsC, nch1 = (nch + 1) / 2;
    const int64_t mid = (nch1 * kBsC < T) ? nch1 * kBsC : T;
    auto nrows = [&](int64_t c) -> int { return (int)((T - c * kBsC < kBsC) ? T - c * kBsC : kBsC); };
    auto iss = [&](int64_t c, int64_t lo, int64_t hi) { rl.issue(c, c >= lo && c < hi); };
    int par = 0;
    // one max-plus step over the exchanged vector x (lane j's value): best_j = max_k (x_k - o + LA[k]),
    // smallest maximising k; returns o = max x (0 if all -inf)
    auto mp_step = [&](float xv, float& best, int& arg, bool& dead) -> float {
        float* xb = xbuf + par * DP;
        par ^= 1;
        xb[j] = xv;
        __syncwarp(gm);
        float v[DP];
        ld_vec<DP>(xb, v);
        float o = tmax<DP>(v);
        dead = !(o > neg_inf());
        if (dead) o = 0.0f;
        // scores v_k + LA_k, the max subtracted once from the winner (D adds fewer than normalising v);
        // smallest maximising k by a select chain (off the recursion's critical path)
        float sc[DP];
#pragma unroll
        for (int k = 0; k < DP; k++) sc[k] = v[k] + LA[k];
        const float bm = tmax<DP>(sc);
        int a = DP - 1;
#pragma unroll
        for (int k = DP - 2; k >= 0; k--) a = (sc[k] == bm) ? k : a;
        arg = a;
        best = bm - o;
        return o;
    };
    double cf = 0.0;  // forward offset: V_t = V~_t + cf
    int64_t zero_t = -1;
    bool bad = false;
    float V = neg_inf();
    // forward max-product with backpointers over chunks [lo, hi) (Algorithm 4 lines 3-6)
    auto fwd_range = [&](int64_t lo, int64_t hi) {
        iss(lo, lo, hi);
        for (int64_t ch = lo; ch < hi; ch++) {
            iss(ch + 1, lo, hi);
            cp_async_wait<1>();
            __syncwarp(gm);
            float* rows = rl.stage(ch);
            const int n = nrows(ch);
            bad |= bs2_prep<DP, true>(rows, mrow, n, D, j, gm);
            for (int i = 0; i < n; i++) {
                const int64_t t = ch * kBsC + i;
                const float w = rows[i * DP + j];
                const float m = mrow[i];
                if (t == 0) {
                    V = lpv + w;
                    cf = (double)m;
                } else {
                    float best;
                    int arg;
                    bool dead;
                    const float o = mp_step(V, best, arg, dead);
                    if (dead && zero_t < 0) zero_t = t - 1;
                    if (act) bp[t * DP + j] = (uint8_t)arg;
                    V = best + w;
                    cf += (double)o + (double)m;
                }
            }
            __syncwarp(gm);
        }
        cp_async_wait<0>();
        __syncwarp(gm);
    };
    // path over steps [s, e) through SMEM-staged pointer chunks: backward (x given at e-1, x_{t-1} =
    // bp_t(x_t)) or forward (x given at s-1, x_t = fp_t(x_{t-1}))
    auto walk = [&](int64_t s, int64_t e, int x, bool backward) {
        for (int64_t q = 0; q < e - s; q += kBsChunk) {
            const int64_t s0 = backward ? ((e - q - kBsChunk > s) ? e - q - kBsChunk : s) : s + q;
            const int64_t e0 = backward ? e - q : ((s + q + kBsChunk < e) ? s + q + kBsChunk : e);
            const int n = (int)(e0 - s0);
            for (int r = j; r < n * DP / 4; r += DP)
                reinterpret_cast<uint32_t*>(sbp)[r] = reinterpret_cast<const uint32_t*>(bp + s0 * DP)[r];
            __syncwarp(gm);
            if (j == 0) {
                if (backward) {
                    for (int i = n - 1; i >= 0; i--) {
                        spath[i] = x;
                        if (s0 + i > 0) x = sbp[i * DP + x];
                    }
                } else {
                    for (int i = 0; i < n; i++) {
                        x = sbp[i * DP + x];
                        spath[i] = x;
                    }
                }
            }
            x = __shfl_sync(gm, x, 0, DP);
            __syncwarp(gm);
            for (int i = j; i < n; i += DP) p.path[base + s0 + i] = spath[i];
            __syncwarp(gm);
        }
    };
    auto vec_argmax = [&](const float* vv, float& o) -> int {
        float v[DP];
        ld_vec<DP>(vv, v);
        o = tmax<DP>(v);
        return first_argmax<DP>(v, o);
    };

    if (live) {
        if (role == 0) {
            fwd_range(0, nch1);
            bad = __any_sync(gm, bad);
            vmeet[g][0][j] = V;
        } else {
            // backward max-product over [mid, T) (Lemma 3's backward recursion): U = V^b_t; forward
            // pointers fp_t(i) = argmax_k (log A(i, k) + w_t(k) + V^b_t(k)) stored at bp[t][i]
            float U = act ? 0.0f : neg_inf();
            double cb = 0.0;
            bool dead_any = false;
            iss(nch - 1, nch1, nch);
            for (int64_t ch = nch - 1; ch >= nch1; ch--) {
                iss(ch - 1, nch1, nch);
                cp_async_wait<1>();
                __syncwarp(gm);
                float* rows = rl.stage(ch);
                const int n = nrows(ch);
                bad |= bs2_prep<DP, true>(rows, mrow, n, D, j, gm);
                for (int i = n - 1; i >= 0; i--) {
                    const int64_t t = ch * kBsC + i;
                    float best;
                    int arg;
                    bool dead;
                    const float o = mp_step(U + rows[i * DP + j], best, arg, dead);
                    dead_any |= dead;
                    if (act) bp[t * DP + j] = (uint8_t)arg;
                    U = act ? best : neg_inf();
                    cb += (double)o + (double)mrow[i];
                }
                __syncwarp(gm);
            }
            cp_async_wait<0>();
            bad = __any_sync(gm, bad);
            vmeet[g][1][j] = U;
            if (j == 0) { cmeet[g] = cb; fmeet[g] = (bad ? 1 : 0) | (dead_any ? 2 : 0); }
        }
    }
    __threadfence_block();
    __syncthreads();  // meet: V^f_{mid-1}, V^b_{mid-1}, the pointers of both halves
    if (!live) return;

    float tot_o;
    int xs;
    {
        float* xb = xbuf + par * DP;
        xb[j] = vmeet[g][0][j] + vmeet[g][1][j];
        __syncwarp(gm);
        xs = vec_argmax(xb, tot_o);
        __syncwarp(gm);
    }
    const bool fallback = !(tot_o > neg_inf()) || (fmeet[g] & 2);
    if (role == 0) {
        const bool bd = bad || (fmeet[g] & 1);
        double lp;
        if (!fallback) {
            lp = (double)tot_o + cf + cmeet[g];
            walk(0, mid, xs, true);
        } else {
            // an impossible step somewhere: the forward pass over the rest locates it (info) and the
            // path is backtracked from argmax V_{T-1} as in the one-warp plan
            fwd_range(nch1, nch);
            float* xb = xbuf + par * DP;
            xb[j] = V;
            __syncwarp(gm);
            float o;
            int x = vec_argmax(xb, o);
            if (!(o > neg_inf())) {
                if (zero_t < 0) zero_t = T - 1;
                o = 0.0f;
                x = 0;
            }
            lp = cf + (double)o;
            __syncwarp(gm);
            walk(0, T, x, true);
        }
        if (j == 0) {
            p.scalar_out[b] = lp;
            int32_t inf = 0;
            if (bd || lp != lp) inf = -1;
            else if (zero_t >= 0) inf = (int32_t)(zero_t + 1);
            if (raw < 1 || raw > p.T) inf = kInfoBadLength;
            p.info[b] = inf;
        }
    } else if (!fallback && mid < T) {
        walk(mid, T, xs, false);
    }
}

// ---------------------------------------------------------------------------- bidirectional smoother,
// warp-specialised: per role (forward / backward) a recursion warp runs only the recursion steps while a
// helper warp streams the chunks in (cp.async), prepares them (row maxima, l = exp(ll - m)) one chunk
// ahead and normalises + stores the finished chunk behind it (filtered / smoothed / kept b_t) -- the
// chunk bookkeeping no longer sits between the recursion's steps (it cost ~0.4 ms of 1.16 at config 4).
// One named barrier per role and chunk (64 threads: the two warps of the role); chunks of kBs3C steps, a
// 3-deep ring (in use / prepared / loading) and a double-buffered output staging.  Lane groups of a warp
// (two sequences at DP = 16) walk their own chunk ranges in lockstep (warp-uniform trip counts).
constexpr int kBs3C = 16;
constexpr int kBs3Threads = 128;
template <int DP> struct Bs3 {
    static constexpr int G = 32 / DP;
    static constexpr int RING = 3 * kBs3C * DP;
    static constexpr int OUTB = (kBs3C + 1) * DP;                 // one staging buffer (row 0 = carry)
    static constexpr int PER = 2 * RING + 2 * OUTB + 2 * kBs3C;   // floats per (role, group)
};
template <int DP>
struct Bs3Ring {
    float* buf;  // [3][kBs3C][DP]
    const float* src;
    int64_t T;
    int D, j;
    bool vec;
    __device__ __forceinline__ float* stage(int64_t c) const { return buf + (size_t)((uint32_t)c % 3u) * kBs3C * DP; }
    __device__ __forceinline__ void issue(int64_t c, bool ok) const {
        if (ok && c >= 0 && c * kBs3C < T) {
            const int64_t r0 = c * kBs3C;
            const int n = (int)((T - r0 < kBs3C) ? T - r0 : kBs3C);
            if (vec) {
                float* dst = stage(c);
                const float* s = src + r0 * D;
                const int Dl = D;
                for_quads<DP>(n, D >> 2, j, [&](int r, int q) { cp_async16(dst + r * DP + 4 * q, s + (int64_t)r * Dl + 4 * q); });
            } else if (j < D) {
                float* dst = stage(c) + j;
                const float* s = src + r0 * D + j;
                for (int r = 0; r < n; r++) cp_async4(dst + r * DP, s + (int64_t)r * D);
            }
        }
        cp_async_commit();
    }
};

template <int DP>
__global__ void __launch_bounds__(kBs3Threads) bs3_smooth_kernel(const BSParams p) {
    using Z = Bs3<DP>;
    constexpr int G = Z::G, RING = Z::RING, OUTB = Z::OUTB, PER = Z::PER;
    extern __shared__ __align__(16) float bsm[];
    __shared__ int s_es[G];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int role = warp & 1, helper = warp >> 1;  // role 0 forward / 1 backward; warp 0,1 recursion, 2,3 helpers
    const int g = lane / DP, j = lane % DP;
    const unsigned gm = bs2_gmask<DP>(g);
    float* region = bsm + (size_t)(role * G + g) * PER;
    float* r0buf = region;            // log_lik chunks -> l (and w = l o b in the backward recursion)
    float* r1buf = region + RING;     // phase 2: forward: kept b_t rows; backward: filtered rows
    float* outb = r1buf + RING;       // [2][1 + C][DP]
    float* mrow = outb + 2 * OUTB;    // [C]
    float* inv = mrow + kBs3C;        // [C]
    const int64_t b = (int64_t)blockIdx.x * G + g;
    int64_t base = 0, raw = 0, T = 0;
    if (b < p.B) T = seq_span(p.offsets, p.T, b, base, raw);
    const bool live = T >= 1;
    if (b < p.B && !live && role == 0 && helper && j == 0) { p.scalar_out[b] = 0.0; p.info[b] = kInfoBadLength; }
    const int D = p.D;
    const bool act = j < D;
    const int64_t nch = (T + kBs3C - 1) / kBs3C, nch1 = (nch + 1) / 2;
    const int64_t mid = (nch1 * kBs3C < T) ? nch1 * kBs3C : T;
    float* filt = p.filtered + base * D;
    float* smo = p.smoothed + base * D;
    float* sb = p.sbeta + (b < p.B ? b : 0) * p.s_rows * D;  // row t - mid
    const bool vec = bs2_vec_ok(p.log_lik, D) && bs2_vec_ok(p.filtered, D) && bs2_vec_ok(p.smoothed, D) &&
                     bs2_vec_ok(p.sbeta, D);
    const Bs3Ring<DP> rl{r0buf, p.log_lik + base * D, T, D, j, vec};
    const Bs3Ring<DP> r1{r1buf, role == 0 ? sb - mid * D : filt, T, D, j, vec};
    auto nrows = [&](int64_t c) -> int { return (int)((T - c * kBs3C < kBs3C) ? T - c * kBs3C : kBs3C); };
    // per phase: this group's chunk count and the chunk of its k-th iteration; trip count = max over the
    // groups of the warp (warp-uniform, the named barrier counts whole warps)
    auto count = [&](int ph) -> int64_t {
        if (!live) return 0;
        return (role == 0) == (ph == 0) ? nch1 : nch - nch1;
    };
    auto chunk_of = [&](int ph, int64_t k) -> int64_t {
        if (role == 0) return ph == 0 ? k : nch1 + k;
        return ph == 0 ? nch - 1 - k : nch1 - 1 - k;
    };
    auto warp_max = [&](int64_t v) -> int64_t {
        if constexpr (G == 2) {
            const int64_t o = __shfl_xor_sync(0xffffffffu, v, 16);
            return v > o ? v : o;
        }
        return v;
    };
    // output buffer of the group's k-th chunk of phase ph: its chunks alternate buffers across both phases
    // (the forward carry a_{t0-1} travels in row 0 of the next buffer)
    auto par_of = [&](int ph, int64_t k) -> int64_t { return (ph == 1 ? count(0) : 0) + k; };
    const unsigned bar_id = 1 + role;
    auto role_bar = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory"); };

    if (!helper) {
        // ============ recursion warp: only the recursion steps
        const float* la = p.log_A + (b < p.B ? b : 0) * p.A_stride;
        float Am[DP];  // forward: column j of A; backward: row j
#pragma unroll
        for (int i = 0; i < DP; i++)
            Am[i] = (act && i < D && live) ? ex2(__ldg(role == 0 ? la + i * D + j : la + j * D + i) * kLog2e) : 0.0f;
        const float piv = (act && live) ? ex2(__ldg(p.log_pi + b * p.pi_stride + j) * kLog2e) : 0.0f;
        int es = 0;
        float bt = act ? 1.0f : 0.0f;  // b_{T-1} = 1
        for (int ph = 0; ph < 2; ph++) {
            const int64_t n_g = count(ph), nk = warp_max(n_g);
            role_bar();  // B_0: chunk 0 of the phase is prepared
            for (int64_t k = 0; k < nk; k++) {
                if (k < n_g) {
                    const int64_t it = par_of(ph, k);  // this group's chunk counter (output buffer parity)
                    const int64_t c = chunk_of(ph, k);
                    float* rows = rl.stage(c);
                    float* out = outb + (it & 1) * OUTB;
                    const int n = nrows(c);
                    if (role == 0) {
                        for (int i = 0; i < n; i++) {
                            const int64_t t = c * kBs3C + i;
                            const float l = rows[i * DP + j];
                            float a;
                            if (t == 0) {
                                a = piv * l;
                            } else {
                                float v[DP];
                                ld_vec<DP>(out + i * DP, v);  // a_{t-1}
                                const float mx = tmax<DP>(v);
                                const float s2 = pow2_inv(mx);
                                es += pow2_inv_log2(mx);
                                float c0 = 0.0f, c1 = 0.0f, c2 = 0.0f, c3 = 0.0f;
#pragma unroll
                                for (int q = 0; q < DP; q += 4) {
                                    c0 = fmaf(v[q], Am[q], c0);
                                    c1 = fmaf(v[q + 1], Am[q + 1], c1);
                                    c2 = fmaf(v[q + 2], Am[q + 2], c2);
                                    c3 = fmaf(v[q + 3], Am[q + 3], c3);
                                }
                                a = ((c0 + c1) + (c2 + c3)) * (l * s2);
                            }
                            out[(i + 1) * DP + j] = a;
                            __syncwarp(gm);
                        }
                        outb[((it + 1) & 1) * OUTB + j] = out[n * DP + j];  // carry a_{t0-1} into the next buffer
                    } else {
                        const float* frows = ph == 1 ? r1.stage(c) : nullptr;
                        for (int i = n - 1; i >= 0; i--) {
                            const int64_t t = c * kBs3C + i;
                            out[(i + 1) * DP + j] = frows ? frows[i * DP + j] * bt : bt;  // gam_t, or b_t
                            rows[i * DP + j] *= bt;                                       // w = l_t o b_t
                            __syncwarp(gm);
                            if (t > 0) {
                                float v[DP];
                                ld_vec<DP>(rows + i * DP, v);
                                const float s2 = pow2_inv(tmax<DP>(v));
                                float c0 = 0.0f, c1 = 0.0f, c2 = 0.0f, c3 = 0.0f;
#pragma unroll
                                for (int q = 0; q < DP; q += 4) {
                                    c0 = fmaf(Am[q], v[q], c0);
                                    c1 = fmaf(Am[q + 1], v[q + 1], c1);
                                    c2 = fmaf(Am[q + 2], v[q + 2], c2);
                                    c3 = fmaf(Am[q + 3], v[q + 3], c3);
                                }
                                bt = ((c0 + c1) + (c2 + c3)) * s2;
                            }
                        }
                    }
                    __syncwarp(gm);
                }
                role_bar();  // B_{k+1}: chunk k staged for the helper, chunk k+1 prepared
            }
            __syncthreads();  // phase boundary (both roles; the helpers flush the last chunk first)
        }
        if (role == 0 && j == 0) s_es[g] = es;
        __syncthreads();
        return;
    }

    // ============ helper warp: loads, preparation one chunk ahead, output one chunk behind
    double msum = 0.0;
    int64_t zero_t = -1;
    bool bad = false;
    float lastsum = 0.0f;
    for (int i = j; i < 2 * RING + 2 * OUTB + 2 * kBs3C; i += DP) region[i] = 0.0f;  // pads stay 0
    __syncwarp(gm);
    auto prep = [&](int ph, int64_t k, int64_t n_g) {
        if (k >= n_g) return;
        const int64_t c = chunk_of(ph, k);
        const int n = nrows(c);
        const bool bd = bs2_prep<DP, false>(rl.stage(c), mrow, n, D, j, gm, role == 0 ? &msum : nullptr);
        if (role == 0) bad |= bd;
    };
    auto flush = [&](int ph, int64_t k, int64_t n_g) {
        if (k < 0 || k >= n_g) return;
        const int64_t c = chunk_of(ph, k);
        const int n = nrows(c);
        float* out = outb + (par_of(ph, k) & 1) * OUTB + DP;
        bool dummy = false;
        float dl;
        if (role == 0) {
            const int z = bs2_flush<DP>(out, n, filt + c * kBs3C * D, D, j, gm, inv, bad, lastsum, vec);
            if (z >= 0 && zero_t < 0) zero_t = c * kBs3C + z;
            if (ph == 1) {  // smoothed = a_t o b_t / sum, in place over the kept b_t rows
                float* brows = r1.stage(c);
                for_quads_c<DP, DP / 4>(n, j, [&](int r, int q) {  // gam_t = a_t o b_t, 16-B quads
                    float4* pb = reinterpret_cast<float4*>(brows + r * DP) + q;
                    const float4 x = *pb, y = reinterpret_cast<const float4*>(out + r * DP)[q];
                    *pb = make_float4(x.x * y.x, x.y * y.y, x.z * y.z, x.w * y.w);
                });
                __syncwarp(gm);
                bs2_flush<DP, false>(brows, n, smo + c * kBs3C * D, D, j, gm, inv, dummy, dl, vec);
            }
        } else {
            float* dst = ph == 0 ? sb + (c * kBs3C - mid) * D : smo + c * kBs3C * D;
            bs2_flush<DP, false>(out, n, dst, D, j, gm, inv, dummy, dl, vec);
        }
    };
    for (int ph = 0; ph < 2; ph++) {
        const int64_t n_g = count(ph), nk = warp_max(n_g);
        const bool two = (ph == 1);  // phase 2 also streams the r1 ring (kept b_t / filtered rows)
        auto load = [&](int64_t k) {
            const bool ok = k >= 0 && k < n_g;
            const int64_t c = ok ? chunk_of(ph, k) : 0;
            rl.issue(c, ok);
            if (two) r1.issue(c, ok); else cp_async_commit();
        };
        load(0);
        load(1);
        cp_async_wait<2>();
        __syncwarp(gm);
        prep(ph, 0, n_g);
        role_bar();  // B_0
        for (int64_t k = 0; k < nk; k++) {
            flush(ph, k - 1, n_g);  // the chunk the recursion finished before B_k
            load(k + 2);                    // into the stage of chunk k-1 (done with above)
            cp_async_wait<2>();
            __syncwarp(gm);
            prep(ph, k + 1, n_g);
            role_bar();  // B_{k+1}
        }
        flush(ph, nk - 1, n_g);
        cp_async_wait<0>();
        __threadfence_block();
        __syncthreads();  // phase boundary
    }
    __syncthreads();  // the recursion warp's exponent sum
    bad = __any_sync(gm, bad);
#pragma unroll
    for (int o = DP / 2; o >= 1; o >>= 1) msum += __shfl_xor_sync(gm, msum, o, DP);  // fixed-order tree
    if (role == 0 && live && j == 0) {
        const double logz = log((double)lastsum) - (double)s_es[g] * (double)kLn2 + msum;
        p.scalar_out[b] = logz;
        int32_t inf = 0;
        if (bad || logz != logz) inf = -1;
        else if (zero_t >= 0) inf = (int32_t)(zero_t + 1);
        if (raw < 1 || raw > p.T) inf = kInfoBadLength;
        p.info[b] = inf;
    }
}

size_t bs_smem(int DP, int op, bool bidir) {
    if (bidir) {
        const size_t per = DP == 16 ? (op == 0 ? Bs3<16>::PER : Bs2<16>::VT_PER)
                                    : (op == 0 ? Bs3<32>::PER : Bs2<32>::VT_PER);
        return per * 4 * 2 * (32 / DP);  // 2 roles x sequences per warp
    }
    const size_t ring = (size_t)kBsStages * kBsC * DP;
    const size_t per = op == 0 ? 2 * ring + (size_t)(kBsC + 1) * DP + 2 * kBsC
                               : ring + 2 * DP + kBsC + kBsChunk + (size_t)kBsChunk * DP / 4;
    return per * 4 * (kBsThreads / 32);
}
// rows of kept b_t per sequence: the second half of the smoother's kBs3C-step chunks (T <= Tmax)
int64_t bs2_beta_rows(int64_t Tmax) {
    const int64_t nch = (Tmax + kBs3C - 1) / kBs3C;
    return (nch / 2) * kBs3C;
}

cudaError_t launch_batchseq(int DP, int op, bool bidir, const BSParams& p, cudaStream_t s) {
    const size_t sm = bs_smem(DP, op, bidir);
    const void* k = nullptr;
    if (bidir) {
        if (DP == 16) k = op == 0 ? (const void*)bs3_smooth_kernel<16> : (const void*)bs2_viterbi_kernel<16>;
        else if (DP == 32) k = op == 0 ? (const void*)bs3_smooth_kernel<32> : (const void*)bs2_viterbi_kernel<32>;
        else return cudaErrorInvalidValue;
        if (cudaError_t e = ensure_smem_optin(k, sm); e != cudaSuccess) return e;
        const unsigned grid = (unsigned)((p.B + 32 / DP - 1) / (32 / DP));  // (forward, backward) roles x 32/DP seqs
        if (DP == 16) {
            if (op == 0) bs3_smooth_kernel<16><<<grid, kBs3Threads, sm, s>>>(p);
            else bs2_viterbi_kernel<16><<<grid, kBs2Threads, sm, s>>>(p);
        } else {
            if (op == 0) bs3_smooth_kernel<32><<<grid, kBs3Threads, sm, s>>>(p);
            else bs2_viterbi_kernel<32><<<grid, kBs2Threads, sm, s>>>(p);
        }
        return cudaGetLastError();
    }
    const unsigned spb = kBsThreads / 32;  // one warp per sequence
    const unsigned grid = (unsigned)((p.B + spb - 1) / spb);
    if (DP == 16) k = op == 0 ? (const void*)bs_smooth_kernel<16> : (const void*)bs_viterbi_kernel<16>;
    else if (DP == 32) k = op == 0 ? (const void*)bs_smooth_kernel<32> : (const void*)bs_viterbi_kernel<32>;
    else return cudaErrorInvalidValue;
    if (cudaError_t e = ensure_smem_optin(k, sm); e != cudaSuccess) return e;
    if (DP == 16) {
        if (op == 0) bs_smooth_kernel<16><<<grid, kBsThreads, sm, s>>>(p);
        else bs_viterbi_kernel<16><<<grid, kBsThreads, sm, s>>>(p);
    } else {
        if (op == 0) bs_smooth_kernel<32><<<grid, kBsThreads, sm, s>>>(p);
        else bs_viterbi_kernel<32><<<grid, kBsThreads, sm, s>>>(p);
    }
    return cudaGetLastError();
}

}  // namespace hmm
