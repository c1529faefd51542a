// hmm_large.cu — parallel-scan HMM smoother and Viterbi for 9 <= D <= 64 (padded to DP in {16,32,64}),
// sm_100a, FP32 CUDA cores.
//
// Same method as hmm_small.cu (block-wise elements of PAPER.md:759-760 scanned with the operators of
// Def. 3 / Def. 5), organised for large D where one element product is a
// DP x DP x DP contraction:
//
//   K1 lg_leaf   one warp per leaf (two half-warp leaves when DP = 16).  Lane owns CPL = DP/32 columns
//                of A in registers; the leaf product P lives in SMEM and is read row by row as warp
//                broadcasts (row r of P.A depends only on row r of P, so rows are updated in place).
//                Per-step exact pow2 (or max-subtract) normalisation.  The block's leaves are then
//                combined by an SMEM tree into the block root.
//   K2 lg_carry  one CTA per sequence: forward (and backward) vector chains through the block roots
//                (D^2 per root, the carries of Thms 1-2 / Props 2-3 at block granularity).
//   K3 lg_sweep  per block: vector chains through its leaves, then per-leaf sequential sweeps
//                (Alg. 1 / Alg. 4 restricted to the leaf) writing filtered/smoothed or backpointers.
//   K4/K5        Viterbi: block end states by composing block backpointer maps, then backtrack.
//   finalize     fixed-order fp64 sum of per-leaf partials -> log Z / log_prob; info.
#include <cfloat>
#include <cstdint>
#include <cstring>

#include "hmm_device.cuh"
#include "hmm_large.h"
#include "hmm_plan.h"

namespace hmm {

cudaError_t launch_large_tc_leaf(const LgParams& p, float* lik, cudaStream_t s);

template <int DP>
struct LG {
    static constexpr int CPL = DP >= 32 ? DP / 32 : 1;  // columns (or rows) per lane
    static constexpr int LPL = DP / CPL;                // lanes per leaf
    static constexpr int LPW = 32 / LPL;                // leaves per warp
    static constexpr int NW = 8;                        // warps per CTA
    static constexpr int NLB = NW * LPW;                // leaves per CTA ("block")
};

template <int LPL>
__device__ __forceinline__ float grp_max(float v) {
#pragma unroll
    for (int o = 1; o < LPL; o <<= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
template <int LPL>
__device__ __forceinline__ float grp_sum(float v) {
#pragma unroll
    for (int o = 1; o < LPL; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float lg_pad(bool mp) { return mp ? neg_inf() : 0.0f; }

__device__ __forceinline__ int og_global_lookup(const LgParams& p, int64_t b, int64_t L, int x, int DP) {
    return p.lmap[((size_t)b * p.NL + L) * DP + x];
}

// A(k, j) for the padded model (exp for sum-product, log for max-product).
__device__ __forceinline__ float lg_A(const LgParams& p, int64_t b, int k, int j, bool mp) {
    if (k >= p.D || j >= p.D) return lg_pad(mp);
    const float la = __ldg(p.log_A + b * p.A_stride + k * p.D + j);
    return mp ? la : ex2(la * kLog2e);
}
__device__ __forceinline__ float lg_pi(const LgParams& p, int64_t b, int j, bool mp) {
    if (j >= p.D) return lg_pad(mp);
    const float lp = __ldg(p.log_pi + b * p.pi_stride + j);
    return mp ? lp : ex2(lp * kLog2e);
}

// Row-wise in-place product of two DP x DP SMEM matrices by one (sub-)leaf group of lanes:
// X <- X (op) Y, where the lanes hold Y's columns in registers (Ycol).  Normalised (pow2 / max).
template <int DP, bool MP>
__device__ void lg_rows_times(float* X, const float (&Ycol)[LG<DP>::CPL][DP], int cl, bool act) {
    constexpr int CPL = LG<DP>::CPL, LPL = LG<DP>::LPL;
    float mx = MP ? neg_inf() : 0.0f;
    for (int r = 0; r < DP; r++) {
        float acc[CPL];
#pragma unroll
        for (int c = 0; c < CPL; c++) acc[c] = MP ? neg_inf() : 0.0f;
#pragma unroll
        for (int k4 = 0; k4 < DP; k4 += 4) {
            const float4 x = *reinterpret_cast<const float4*>(X + r * DP + k4);
#pragma unroll
            for (int c = 0; c < CPL; c++) {
                if constexpr (MP) {
                    acc[c] = fmaxf(acc[c], max3(x.x + Ycol[c][k4], x.y + Ycol[c][k4 + 1],
                                                fmaxf(x.z + Ycol[c][k4 + 2], x.w + Ycol[c][k4 + 3])));
                } else {
                    acc[c] = fmaf(x.x, Ycol[c][k4], acc[c]);
                    acc[c] = fmaf(x.y, Ycol[c][k4 + 1], acc[c]);
                    acc[c] = fmaf(x.z, Ycol[c][k4 + 2], acc[c]);
                    acc[c] = fmaf(x.w, Ycol[c][k4 + 3], acc[c]);
                }
            }
        }
        __syncwarp();
        if (act) {
#pragma unroll
            for (int c = 0; c < CPL; c++) {
                X[r * DP + cl * CPL + c] = acc[c];
                mx = fmaxf(mx, acc[c]);
            }
        }
        __syncwarp();
    }
    mx = grp_max<LPL>(mx);
    if (act) {
        for (int r = 0; r < DP; r++) {
#pragma unroll
            for (int c = 0; c < CPL; c++) {
                float& v = X[r * DP + cl * CPL + c];
                if constexpr (MP) {
                    if (mx > neg_inf()) v -= mx;
                } else {
                    v *= pow2_inv(mx);
                }
            }
        }
    }
    __syncwarp();
}

// ------------------------------------------------------------------------------------------- K1
template <int DP, int OP>
__global__ void __launch_bounds__(256) lg_leaf_kernel(const LgParams p) {
    using C = LG<DP>;
    constexpr int CPL = C::CPL, LPL = C::LPL, LPW = C::LPW, NLB = C::NLB;
    constexpr bool MP = (OP == 1);
    extern __shared__ __align__(128) uint8_t smem[];
    float* sm = reinterpret_cast<float*>(smem);
    const int64_t b = blockIdx.y;
    const int blk = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sub = lane / LPL, cl = lane % LPL;
    const int lidx = warp * LPW + sub;                    // leaf index inside the block
    const int64_t L = (int64_t)blk * NLB + lidx;          // leaf index inside the sequence
    float* Pm = sm + (size_t)lidx * DP * DP;
    int64_t sbase, T_raw;  // packed first row / length of sequence b (varlen batches, f4)
    const int64_t T = seq_span(p.offsets, p.T, b, sbase, T_raw);
    const int64_t t0 = L * p.SL;
    auto leaf_len = [&](int64_t LL) -> int {
        const int64_t a = LL * p.SL;
        if (LL >= p.NL || a >= T) return 0;
        return (int)((T - a < p.SL) ? T - a : p.SL);
    };
    const int n = leaf_len(L);
    int nmax = n;
#pragma unroll
    for (int o = LPL; o < 32; o <<= 1) nmax = max(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));

    if (MP || !p.tc) {
        float Acol[CPL][DP], pv[CPL];
    #pragma unroll
        for (int c = 0; c < CPL; c++) {
            const int j = cl * CPL + c;
    #pragma unroll
            for (int k = 0; k < DP; k++) Acol[c][k] = lg_A(p, b, k, j, MP);
            pv[c] = lg_pi(p, b, j, MP);
        }
        constexpr bool PK = (CPL == 1);           // packed row pairs (DP = 16, 32; see the loop)
        constexpr bool PC = (CPL == 2 && MP);     // packed column pairs (max-product, DP = 64)
        float2 A2[(PK || PC) ? DP : 1];
        if constexpr (PK) {
    #pragma unroll
            for (int k = 0; k < DP; k++) A2[k] = make_float2(Acol[0][k], Acol[0][k]);
        }
        if constexpr (PC) {
    #pragma unroll
            for (int k = 0; k < DP; k++) A2[k] = make_float2(Acol[0][k], Acol[1][k]);
        }
        const float* ll = p.log_lik + (size_t)sbase * p.D;
        bool bad = false;
        float s = MP ? 0.0f : 1.0f;  // pending normalisation (scale / offset) from the previous step
        float chk = 0.0f;
        for (int i = 0; i < nmax; i++) {
            const bool act = i < n;
            const int64_t t = t0 + i;
            float v[CPL], l[CPL];
    #pragma unroll
            for (int c = 0; c < CPL; c++) {
                const int j = cl * CPL + c;
                v[c] = (act && j < p.D) ? __ldg(ll + t * p.D + j) : neg_inf();
            }
            float m = v[0];
    #pragma unroll
            for (int c = 1; c < CPL; c++) m = fmaxf(m, v[c]);
            m = grp_max<LPL>(m);
            if (!(m > neg_inf())) m = 0.0f;
    #pragma unroll
            for (int c = 0; c < CPL; c++) {
                if constexpr (MP) {
                    l[c] = v[c] - m;
                    chk += l[c];
                } else {
                    l[c] = ex2((v[c] - m) * kLog2e);
                }
            }
            if constexpr (PK) {
                // DP = 16, one column per lane: P kept with row pairs interleaved, element (r, j) at
                // Pm[(r/2)*2DP + 2j + r%2], so one LDS.128 yields (P(r,k), P(r+1,k)) and (P(r,k+1),
                // P(r+1,k+1)) and each FFMA2 / FADD2 updates two rows of the lane's column with the
                // duplicated A(k, j): the same multiply-adds as the scalar loop in half the issue slots
                // (the max-product adds keep their operands, so its values are bit-identical).
                constexpr int NRP = DP / 2;
                if (i == 0) {
                    if (act) {
    #pragma unroll
                        for (int rp = 0; rp < NRP; rp++) {
                            const float a0 = (p.t_base + t == 0) ? pv[0] : Acol[0][2 * rp];
                            const float a1 = (p.t_base + t == 0) ? pv[0] : Acol[0][2 * rp + 1];
                            *reinterpret_cast<float2*>(Pm + rp * 2 * DP + 2 * cl) =
                                MP ? make_float2(a0 + l[0], a1 + l[0]) : make_float2(a0 * l[0], a1 * l[0]);
                        }
                    }
                    __syncwarp();
                } else {
                    float2 acc[NRP];
    #pragma unroll
                    for (int rp = 0; rp < NRP; rp++) acc[rp] = MP ? make_float2(neg_inf(), neg_inf()) : make_float2(0.0f, 0.0f);
    #pragma unroll
                    for (int rp = 0; rp < NRP; rp++) {
    #pragma unroll
                        for (int k = 0; k < DP; k += 2) {
                            const float4 x = *reinterpret_cast<const float4*>(Pm + rp * 2 * DP + 2 * k);
                            if constexpr (MP) {
                                const float2 s0 = __fadd2_rn(make_float2(x.x, x.y), A2[k]);
                                const float2 s1 = __fadd2_rn(make_float2(x.z, x.w), A2[k + 1]);
                                acc[rp] = make_float2(max3(acc[rp].x, s0.x, s1.x), max3(acc[rp].y, s0.y, s1.y));
                            } else {
                                acc[rp] = __ffma2_rn(make_float2(x.x, x.y), A2[k], acc[rp]);
                                acc[rp] = __ffma2_rn(make_float2(x.z, x.w), A2[k + 1], acc[rp]);
                            }
                        }
                    }
                    __syncwarp();
                    float mx = MP ? neg_inf() : 0.0f;
                    if (act) {
                        const float f = MP ? (l[0] - s) : (l[0] * s);
                        const float2 f2 = make_float2(f, f);
    #pragma unroll
                        for (int rp = 0; rp < NRP; rp++) {
                            const float2 val = MP ? __fadd2_rn(acc[rp], f2) : __fmul2_rn(acc[rp], f2);
                            *reinterpret_cast<float2*>(Pm + rp * 2 * DP + 2 * cl) = val;
                            mx = max3(mx, val.x, val.y);
                        }
                    }
                    __syncwarp();
                    mx = grp_max<LPL>(mx);
                    if constexpr (MP) {
                        s = (mx > neg_inf()) ? mx : 0.0f;
                    } else {
                        s = pow2_inv(mx);
                    }
                }
                continue;
            }
            if (i == 0) {
                if (act) {
    #pragma unroll
                    for (int r = 0; r < DP; r++)
    #pragma unroll
                        for (int c = 0; c < CPL; c++) {
                            const float a = (p.t_base + t == 0) ? pv[c] : Acol[c][r];
                            Pm[r * DP + cl * CPL + c] = MP ? a + l[c] : a * l[c];
                        }
                }
                __syncwarp();
            } else {
                float mx = MP ? neg_inf() : 0.0f;
                // rows in groups of RG: row r of P psi depends only on row r of P, so a group is read,
                // computed with RG independent accumulator chains, then written back in place
                constexpr int RG = (CPL == 1) ? (DP < 32 ? DP : 16) : 8;
                for (int r0 = 0; r0 < DP; r0 += RG) {
                    float acc[RG][CPL];
    #pragma unroll
                    for (int rr = 0; rr < RG; rr++)
    #pragma unroll
                        for (int c = 0; c < CPL; c++) acc[rr][c] = MP ? neg_inf() : 0.0f;
    #pragma unroll
                    for (int rr = 0; rr < RG; rr++) {
    #pragma unroll
                        for (int k4 = 0; k4 < DP; k4 += 4) {
                            const float4 x = *reinterpret_cast<const float4*>(Pm + (r0 + rr) * DP + k4);
    #pragma unroll
                            for (int c = 0; c < CPL; c++) {
                                if constexpr (PC) {
                                    // the lane's two columns as one FADD2 per k (scalar P(r,k) broadcast),
                                    // maxima by FMNMX3: same sums as the scalar form, bit-identical
                                    if (c == 0) {
                                        const float2 s0 = __fadd2_rn(make_float2(x.x, x.x), A2[k4]);
                                        const float2 s1 = __fadd2_rn(make_float2(x.y, x.y), A2[k4 + 1]);
                                        const float2 s2 = __fadd2_rn(make_float2(x.z, x.z), A2[k4 + 2]);
                                        const float2 s3 = __fadd2_rn(make_float2(x.w, x.w), A2[k4 + 3]);
                                        acc[rr][0] = max3(max3(acc[rr][0], s0.x, s1.x), s2.x, s3.x);
                                        acc[rr][1] = max3(max3(acc[rr][1], s0.y, s1.y), s2.y, s3.y);
                                    }
                                } else if constexpr (MP) {
                                    acc[rr][c] = fmaxf(acc[rr][c], max3(x.x + Acol[c][k4], x.y + Acol[c][k4 + 1],
                                                                        fmaxf(x.z + Acol[c][k4 + 2], x.w + Acol[c][k4 + 3])));
                                } else {
                                    acc[rr][c] = fmaf(x.x, Acol[c][k4], acc[rr][c]);
                                    acc[rr][c] = fmaf(x.y, Acol[c][k4 + 1], acc[rr][c]);
                                    acc[rr][c] = fmaf(x.z, Acol[c][k4 + 2], acc[rr][c]);
                                    acc[rr][c] = fmaf(x.w, Acol[c][k4 + 3], acc[rr][c]);
                                }
                            }
                        }
                    }
                    __syncwarp();
                    if (act) {
    #pragma unroll
                        for (int rr = 0; rr < RG; rr++)
    #pragma unroll
                            for (int c = 0; c < CPL; c++) {
                                const float val = MP ? acc[rr][c] + (l[c] - s) : acc[rr][c] * (l[c] * s);
                                Pm[(r0 + rr) * DP + cl * CPL + c] = val;
                                mx = fmaxf(mx, val);
                            }
                    }
                    __syncwarp();
                }
                mx = grp_max<LPL>(mx);
                if constexpr (MP) {
                    s = (mx > neg_inf()) ? mx : 0.0f;
                } else {
                    s = pow2_inv(mx);
                }
            }
        }
        if constexpr (PK) {  // back to row-major (each lane moves its own column)
            if (nmax > 0) {
                float colv[DP];
    #pragma unroll
                for (int rp = 0; rp < DP / 2; rp++) {
                    const float2 v2 = *reinterpret_cast<const float2*>(Pm + rp * 2 * DP + 2 * cl);
                    colv[2 * rp] = v2.x;
                    colv[2 * rp + 1] = v2.y;
                }
                __syncwarp();
    #pragma unroll
                for (int r = 0; r < DP; r++) Pm[r * DP + cl] = colv[r];
                __syncwarp();
            }
        }
        // final normalisation and NaN check, then write the leaf aggregate (reductions warp-uniform: the
        // two half-warp leaves of DP = 16 may differ in length)
        float mx = MP ? neg_inf() : 0.0f;
        float sum = 0.0f;
        if (n > 0) {
            for (int r = 0; r < DP; r++)
    #pragma unroll
                for (int c = 0; c < CPL; c++) {
                    mx = fmaxf(mx, Pm[r * DP + cl * CPL + c]);
                    sum += Pm[r * DP + cl * CPL + c];
                }
        }
        mx = grp_max<LPL>(mx);
        if (n > 0) {
            if constexpr (!MP) bad |= (sum != sum);
            float* dst = p.leafagg + ((size_t)b * p.NL + L) * DP * DP;
            for (int r = 0; r < DP; r++)
    #pragma unroll
                for (int c = 0; c < CPL; c++) {
                    float& x = Pm[r * DP + cl * CPL + c];
                    if constexpr (MP) {
                        if (mx > neg_inf()) x -= mx;
                    } else {
                        x *= pow2_inv(mx);
                    }
                    dst[r * DP + cl * CPL + c] = x;
                }
        } else {
            // an empty leaf (past the end of a shorter sequence of a varlen batch) is the identity
            // element; the sweep's leaf chains read it back from the workspace
            float* dst = (L < p.NL) ? p.leafagg + ((size_t)b * p.NL + L) * DP * DP : nullptr;
            for (int r = 0; r < DP; r++)
    #pragma unroll
                for (int c = 0; c < CPL; c++) {
                    const int j = cl * CPL + c;
                    const float v = (r == j) ? (MP ? 0.0f : 1.0f) : lg_pad(MP);
                    Pm[r * DP + j] = v;
                    if (dst) dst[r * DP + j] = v;
                }
        }
        if constexpr (MP) bad |= (chk != chk);
        if (bad) atomicOr(reinterpret_cast<uint32_t*>(p.ws_sync + b * 64) + 8, 1u);
    } else {
        // leaf products computed by the tensor-core kernel (hmm_large_tc.cu): load them for the tree
        const float* srcm = p.leafagg + ((size_t)b * p.NL + L) * DP * DP;
        for (int r = 0; r < DP; r++)
#pragma unroll
            for (int c = 0; c < CPL; c++) {
                const int j = cl * CPL + c;
                Pm[r * DP + j] = (L < p.NL) ? __ldcg(srcm + r * DP + j) : ((r == j) ? 1.0f : 0.0f);
            }
    }
    __syncthreads();

    // block root: ordered tree over the NLB leaf buffers (products by leaf lane-groups)
    for (int stride = 1; stride < NLB; stride <<= 1) {
        const bool lead = (lidx % (2 * stride)) == 0 && lidx + stride < NLB;
        const bool any = __any_sync(0xffffffffu, lead);
        if (any) {
            float Ycol[CPL][DP];
            const float* Y = sm + (size_t)(lead ? lidx + stride : lidx) * DP * DP;
#pragma unroll
            for (int c = 0; c < CPL; c++)
#pragma unroll
                for (int k = 0; k < DP; k++) Ycol[c][k] = Y[k * DP + cl * CPL + c];
            __syncwarp();
            lg_rows_times<DP, MP>(Pm, Ycol, cl, lead);
        }
        __syncthreads();
    }
    if (lidx == 0) {
        float* dst = p.groot + ((size_t)b * p.NB + blk) * DP * DP;
        for (int r = 0; r < DP; r++)
#pragma unroll
            for (int c = 0; c < CPL; c++) dst[r * DP + cl * CPL + c] = Pm[r * DP + cl * CPL + c];
    }
}

// ------------------------------------------------------------------------------------------- K2
// Vector chains through a few matrices (one warp each; the leaf carries inside a block, K3).  Lane
// owns output columns / rows.
template <int DP, bool MP>
__device__ void lg_chain_fwd(const float* mats, int64_t nm, const float* v0, float* out /*[nm][DP]*/, float* vs) {
    constexpr int Q = DP >= 32 ? DP / 32 : 1;
    const int lane = threadIdx.x & 31;
    const bool act = lane * Q < DP;
    if (act)
        for (int q = 0; q < Q; q++) vs[lane * Q + q] = v0[lane * Q + q];
    __syncwarp();
    for (int64_t i = 0; i < nm; i++) {
        if (act)
            for (int q = 0; q < Q; q++) out[i * DP + lane * Q + q] = vs[lane * Q + q];
        const float* M = mats + (size_t)i * DP * DP;
        float y[Q];
#pragma unroll
        for (int q = 0; q < Q; q++) y[q] = MP ? neg_inf() : 0.0f;
        if (act) {
            for (int k = 0; k < DP; k++) {
                const float vk = vs[k];
#pragma unroll
                for (int q = 0; q < Q; q++) {
                    const float mkj = __ldcg(M + (size_t)k * DP + lane * Q + q);
                    y[q] = MP ? fmaxf(y[q], vk + mkj) : fmaf(vk, mkj, y[q]);
                }
            }
        }
        float m = y[0];
#pragma unroll
        for (int q = 1; q < Q; q++) m = fmaxf(m, y[q]);
        m = grp_max<32>(act ? m : (MP ? neg_inf() : 0.0f));
        __syncwarp();
        if (act)
            for (int q = 0; q < Q; q++) vs[lane * Q + q] = MP ? ((m > neg_inf()) ? y[q] - m : y[q]) : y[q] * pow2_inv(m);
        __syncwarp();
    }
}
template <int DP>
__device__ void lg_chain_bwd(const float* mats, int64_t nm, const float* w0, float* out, float* ws) {
    constexpr int Q = DP >= 32 ? DP / 32 : 1;
    const int lane = threadIdx.x & 31;
    const bool act = lane * Q < DP;
    if (act)
        for (int q = 0; q < Q; q++) ws[lane * Q + q] = w0[lane * Q + q];
    __syncwarp();
    for (int64_t i = nm - 1; i >= 0; i--) {
        if (act)
            for (int q = 0; q < Q; q++) out[i * DP + lane * Q + q] = ws[lane * Q + q];
        const float* M = mats + (size_t)i * DP * DP;
        float y[Q];
#pragma unroll
        for (int q = 0; q < Q; q++) y[q] = 0.0f;
        if (act) {
#pragma unroll
            for (int q = 0; q < Q; q++) {
                const float* row = M + (size_t)(lane * Q + q) * DP;
                for (int j = 0; j < DP; j++) y[q] = fmaf(__ldcg(row + j), ws[j], y[q]);
            }
        }
        float m = y[0];
#pragma unroll
        for (int q = 1; q < Q; q++) m = fmaxf(m, y[q]);
        m = grp_max<32>(act ? m : 0.0f);
        __syncwarp();
        if (act)
            for (int q = 0; q < Q; q++) ws[lane * Q + q] = y[q] * pow2_inv(m);
        __syncwarp();
    }
}

// Vector chains through the NB block roots of a sequence (the carries of Thms 1-2 / Props 2-3 at
// block granularity): grid (B, 2) -- y = 0 forward (v <- v (op) R_i), y = 1 backward (w <- R_i w,
// sum-product only).  The chain is serial, so the roots stream through an NS-deep cp.async ring
// (16-B chunks XOR-swizzled by row: both the column reads of the forward step and the row reads of
// the backward step are bank-conflict-free) and every step is pure SMEM math on 64 threads.
// Carry chain arguments: the chain runs over `roots` (n per sequence, `rstride` floats apart per
// sequence); CTA (x = b * ng + g, y = dir) covers roots [g gs, min((g+1) gs, n)) starting from the entering
// vector init_pre[b][g] / init_suf[b][g] (null: the boundary vector: 1 / 0 for max-plus), and writes the
// carry entering every root to out_pre / out_suf ([b][root][DP]).
struct LgChain {
    const float* roots;
    int64_t n, rstride, gs, ng;
    const float* init_pre;
    const float* init_suf;
    float* out_pre;
    float* out_suf;
};

template <int DP, int OP>
__global__ void __launch_bounds__(64) lg_carry_kernel(const LgParams p, const LgChain ch) {
    constexpr bool MP = (OP == 1);
    constexpr int NS = 6;                 // ring depth (roots in flight)
    constexpr int CH = DP / 4;            // 16-B chunks per row
    extern __shared__ __align__(16) float ring[];  // [NS][DP*DP]
    __shared__ float vec[DP];
    __shared__ float red[2];
    const int64_t b = blockIdx.x / ch.ng, g = blockIdx.x % ch.ng;
    const bool fwd = blockIdx.y == 0;
    if (!fwd && MP) return;
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t lo = g * ch.gs, hi = (lo + ch.gs < ch.n) ? lo + ch.gs : ch.n;
    const int64_t NB = hi - lo;
    if (NB <= 0) return;
    const float* roots = ch.roots + (size_t)b * ch.rstride + (size_t)lo * DP * DP;
    float* out = (fwd ? ch.out_pre : ch.out_suf) + ((size_t)b * ch.n + lo) * DP;
    const float* init = fwd ? ch.init_pre : ch.init_suf;
    auto sw = [&](int r, int c) -> int { return r * DP + ((c ^ (r & (CH - 1))) << 2); };  // chunk c of row r
    auto load = [&](int64_t i, int st) {
        if (i >= 0 && i < NB) {
            const float* src = roots + (size_t)i * DP * DP;
            float* dst = ring + (size_t)st * DP * DP;
            for (int q = tid; q < DP * CH; q += 64) {
                const int r = q / CH, c = q % CH;
                cp_async16(dst + sw(r, c), src + r * DP + 4 * c);
            }
        }
        cp_async_commit();
    };
    for (int j = tid; j < DP; j += 64)
        vec[j] = init ? init[((size_t)b * ch.ng + g) * DP + j] : (MP ? 0.0f : 1.0f);
    for (int s = 0; s < NS - 1; s++) load(fwd ? s : NB - 1 - s, s);
    __syncthreads();
    for (int64_t it = 0; it < NB; it++) {
        const int64_t i = fwd ? it : NB - 1 - it;
        load(fwd ? it + NS - 1 : NB - 1 - (it + NS - 1), (int)((it + NS - 1) % NS));
        cp_async_wait<NS - 1>();
        __syncthreads();
        const float* M = ring + (size_t)(it % NS) * DP * DP;
        float y = MP ? neg_inf() : 0.0f;
        if (tid < DP) {
            out[(size_t)i * DP + tid] = vec[tid];  // the carry entering root i
            const int c = tid >> 2, w = tid & 3;
            // four independent partial accumulators: the serial chain is latency-bound
            float y4[4] = {y, y, y, y};
            if (fwd) {
#pragma unroll 16
                for (int k = 0; k < DP; k++) {
                    const float mk = M[sw(k, c) + w];
                    y4[k & 3] = MP ? fmaxf(y4[k & 3], vec[k] + mk) : fmaf(vec[k], mk, y4[k & 3]);
                }
            } else {
#pragma unroll 4
                for (int cc = 0; cc < CH; cc++) {
                    const float4 m4 = *reinterpret_cast<const float4*>(M + sw(tid, cc));
                    y4[0] = fmaf(m4.x, vec[4 * cc], y4[0]);
                    y4[1] = fmaf(m4.y, vec[4 * cc + 1], y4[1]);
                    y4[2] = fmaf(m4.z, vec[4 * cc + 2], y4[2]);
                    y4[3] = fmaf(m4.w, vec[4 * cc + 3], y4[3]);
                }
            }
            y = MP ? fmaxf(fmaxf(y4[0], y4[1]), fmaxf(y4[2], y4[3])) : (y4[0] + y4[1]) + (y4[2] + y4[3]);
        }
        float m = (tid < DP) ? y : (MP ? neg_inf() : 0.0f);
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) red[tid >> 5] = m;
        __syncthreads();
        m = fmaxf(red[0], red[1]);
        if (tid < DP) vec[tid] = MP ? ((m > neg_inf()) ? y - m : y) : y * pow2_inv(m);
        // (the next iteration's barrier orders these writes before the reads)
    }
}

// Group products for the two-level carry (long root chains): group g of a sequence = block roots
// [g KG, min((g+1) KG, NB)), multiplied in order (Def. 3 matrix product / Def. 5 max-plus product) and
// renormalised after every product; one CTA of 256 threads per group, thread = 4 x 4 output tile,
// roots double-buffered through SMEM by cp.async.  The carry chain then runs over NB / KG group
// products, and the per-block carries inside a group from the group's carry.
template <int DP, int OP>
__global__ void __launch_bounds__(256) lg_group_kernel(const LgParams p, const float* groot, int64_t NR, int64_t KG,
                                                       int64_t NG, float* gprod) {
    constexpr bool MP = (OP == 1);
    constexpr int TR = DP / 16;  // output rows per thread (DP = 64: 4; 32: 2; 16: 1)
    extern __shared__ __align__(16) float gsm[];  // C [DP][DP], R[2][DP][DP]
    __shared__ float gred[8];
    float* C = gsm;
    const int64_t b = blockIdx.y, g = blockIdx.x;
    const int64_t lo = g * KG, hi = (lo + KG < NR) ? lo + KG : NR;
    const int tid = threadIdx.x;
    const int r0 = (tid / 16) * TR, c0 = (tid % 16) * (DP / 16);
    constexpr int TC = DP / 16;  // output columns per thread
    const float* roots = groot + (size_t)b * NR * DP * DP;
    auto load = [&](int64_t i, float* dst) {
        if (i < hi) {
            const float* src = roots + (size_t)i * DP * DP;
            for (int q = tid; q < DP * DP / 4; q += 256) cp_async16(dst + 4 * q, src + 4 * q);
        }
        cp_async_commit();
    };
    load(lo, C);
    load(lo + 1, gsm + DP * DP);
    for (int64_t i = lo + 1; i < hi; i++) {
        float* R = gsm + (size_t)(1 + ((i - lo - 1) & 1)) * DP * DP;
        load(i + 1, gsm + (size_t)(1 + ((i - lo) & 1)) * DP * DP);
        cp_async_wait<1>();
        __syncthreads();
        float acc[TR][TC];
#pragma unroll
        for (int r = 0; r < TR; r++)
#pragma unroll
            for (int c = 0; c < TC; c++) acc[r][c] = MP ? neg_inf() : 0.0f;
#pragma unroll 8
        for (int k = 0; k < DP; k++) {
            float a[TR], bb[TC];
#pragma unroll
            for (int r = 0; r < TR; r++) a[r] = C[(r0 + r) * DP + k];
#pragma unroll
            for (int c = 0; c < TC; c++) bb[c] = R[k * DP + c0 + c];
#pragma unroll
            for (int r = 0; r < TR; r++)
#pragma unroll
                for (int c = 0; c < TC; c++)
                    acc[r][c] = MP ? fmaxf(acc[r][c], a[r] + bb[c]) : fmaf(a[r], bb[c], acc[r][c]);
        }
        float m = acc[0][0];
#pragma unroll
        for (int r = 0; r < TR; r++)
#pragma unroll
            for (int c = 0; c < TC; c++) m = fmaxf(m, acc[r][c]);
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if ((tid & 31) == 0) gred[tid >> 5] = m;
        __syncthreads();  // every thread has read C and R; the warp maxima are in place
        m = gred[0];
#pragma unroll
        for (int w = 1; w < 8; w++) m = fmaxf(m, gred[w]);
        const float sc = MP ? 0.0f : pow2_inv(m);
#pragma unroll
        for (int r = 0; r < TR; r++)
#pragma unroll
            for (int c = 0; c < TC; c++)
                C[(r0 + r) * DP + c0 + c] = MP ? ((m > neg_inf()) ? acc[r][c] - m : acc[r][c]) : acc[r][c] * sc;
        __syncthreads();
    }
    cp_async_wait<0>();
    __syncthreads();
    float* dst = gprod + ((size_t)b * NG + g) * DP * DP;
    for (int q = tid; q < DP * DP; q += 256) dst[q] = C[q];
}

// ------------------------------------------------------------------------------------------- K3
template <int DP, int OP>
__global__ void __launch_bounds__(256) lg_sweep_kernel(const LgParams p) {
    using C = LG<DP>;
    constexpr int CPL = C::CPL, LPL = C::LPL, LPW = C::LPW, NLB = C::NLB;
    constexpr bool MP = (OP == 1);
    extern __shared__ __align__(128) uint8_t smem[];
    float* lpre = reinterpret_cast<float*>(smem);          // [NLB][DP]
    float* lsuf = lpre + NLB * DP;                          // [NLB][DP]
    float* vec = lsuf + NLB * DP;                           // [NLB][DP] per-leaf broadcast vector
    float* cw = vec + NLB * DP;                             // [2][DP] chain scratch
    uint8_t* orig = reinterpret_cast<uint8_t*>(cw + 2 * DP);  // [NLB][DP] Viterbi origin maps
    const int64_t b = blockIdx.y;
    const int blk = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sub = lane / LPL, cl = lane % LPL;
    const int lidx = warp * LPW + sub;
    const int64_t L = (int64_t)blk * NLB + lidx;
    int64_t sbase, T_raw;  // packed first row / length of sequence b (varlen batches, f4)
    const int64_t T = seq_span(p.offsets, p.T, b, sbase, T_raw);
    const int D = p.D;
    const float* leafs = p.leafagg + ((size_t)b * p.NL + (size_t)blk * NLB) * DP * DP;
    int nleaf = NLB;  // leaves of this block that exist
    if ((int64_t)blk * NLB + nleaf > p.NL) nleaf = (int)(p.NL - (int64_t)blk * NLB);
    // leaf carries: chains through this block's leaves, from the block carries
    if (warp == 0) {
        lg_chain_fwd<DP, MP>(leafs, nleaf, p.bpre + ((size_t)b * p.NB + blk) * DP, lpre, cw);
    } else if (warp == 1 && !MP) {
        lg_chain_bwd<DP>(leafs, nleaf, p.bsuf + ((size_t)b * p.NB + blk) * DP, lsuf, cw + DP);
    }
    __syncthreads();
    int n = 0;
    if (L < p.NL) {
        const int64_t a = L * p.SL;
        n = (a < T) ? (int)((T - a < p.SL) ? T - a : p.SL) : 0;
    }
    int nmax = n;
#pragma unroll
    for (int o = LPL; o < 32; o <<= 1) nmax = max(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
    const int64_t t0 = L * p.SL;
    const float* ll = p.log_lik + (size_t)sbase * D;
    float* vv = vec + lidx * DP;
    uint32_t* sync = reinterpret_cast<uint32_t*>(p.ws_sync + b * 64);
    unsigned long long* zero_code = reinterpret_cast<unsigned long long*>(sync + 4);
    double part = 0.0;
    int64_t zero_t = INT64_MAX;

    if constexpr (!MP) {
        // ---------------- forward filter over the leaf (lane owns CPL columns; A columns in regs)
        float Acol[CPL][DP], pv[CPL];
#pragma unroll
        for (int c = 0; c < CPL; c++) {
#pragma unroll
            for (int k = 0; k < DP; k++) Acol[c][k] = lg_A(p, b, k, cl * CPL + c, false);
            pv[c] = lg_pi(p, b, cl * CPL + c, false);
        }
        float a_own[CPL];
        {
            float s = 0.0f;
#pragma unroll
            for (int c = 0; c < CPL; c++) s += lpre[lidx * DP + cl * CPL + c];
            s = grp_sum<LPL>(s);
            const float r = (s > 0.0f) ? 1.0f / s : 0.0f;
#pragma unroll
            for (int c = 0; c < CPL; c++) {
                a_own[c] = lpre[lidx * DP + cl * CPL + c] * r;
                vv[cl * CPL + c] = a_own[c];
            }
        }
        __syncwarp();
        float rprod = 1.0f;
        int rexp = 0;
        double msum = 0.0;
        float* filt = p.filtered;
        // the log-likelihood row of step i+1 is loaded during step i: the serial per-step chain never
        // waits on global memory
        auto ld_ll = [&](int i, float* v) {
#pragma unroll
            for (int c = 0; c < CPL; c++) {
                const int j = cl * CPL + c;
                v[c] = (i >= 0 && i < n && j < D) ? __ldg(ll + (t0 + i) * D + j) : neg_inf();
            }
        };
        float vnext[CPL];
        ld_ll(0, vnext);
        for (int i = 0; i < nmax; i++) {
            const bool act = i < n;
            const int64_t t = t0 + i;
            float v[CPL], l[CPL], ah[CPL];
#pragma unroll
            for (int c = 0; c < CPL; c++) v[c] = vnext[c];
            ld_ll(i + 1, vnext);
            float m = v[0];
#pragma unroll
            for (int c = 1; c < CPL; c++) m = fmaxf(m, v[c]);
            m = grp_max<LPL>(m);
            if (m > neg_inf()) msum += (cl == 0 && act) ? (double)m : 0.0;
            else m = 0.0f;
#pragma unroll
            for (int c = 0; c < CPL; c++) {
                l[c] = ex2((v[c] - m) * kLog2e);
                ah[c] = 0.0f;
            }
            if (p.t_base + t == 0) {
#pragma unroll
                for (int c = 0; c < CPL; c++) ah[c] = pv[c] * l[c];
            } else {
                // four partial sums per output: the recursion is latency-bound, and a single
                // DP-long FMA chain per output was its critical path
                float q[CPL][4];
#pragma unroll
                for (int c = 0; c < CPL; c++) q[c][0] = q[c][1] = q[c][2] = q[c][3] = 0.0f;
#pragma unroll
                for (int k4 = 0; k4 < DP; k4 += 4) {
                    const float4 x = *reinterpret_cast<const float4*>(vv + k4);
#pragma unroll
                    for (int c = 0; c < CPL; c++) {
                        q[c][0] = fmaf(x.x, Acol[c][k4], q[c][0]);
                        q[c][1] = fmaf(x.y, Acol[c][k4 + 1], q[c][1]);
                        q[c][2] = fmaf(x.z, Acol[c][k4 + 2], q[c][2]);
                        q[c][3] = fmaf(x.w, Acol[c][k4 + 3], q[c][3]);
                    }
                }
#pragma unroll
                for (int c = 0; c < CPL; c++) ah[c] = ((q[c][0] + q[c][1]) + (q[c][2] + q[c][3])) * l[c];
            }
            float cs = 0.0f;
#pragma unroll
            for (int c = 0; c < CPL; c++) cs += ah[c];
            cs = grp_sum<LPL>(cs);
            if (act && !(cs > 0.0f) && p.t_base + t < zero_t) zero_t = p.t_base + t;
            const float r = rcp(cs);
            __syncwarp();
            if (act) {  // a shorter half-warp leaf keeps its final state while its partner runs on
#pragma unroll
                for (int c = 0; c < CPL; c++) {
                    a_own[c] = ah[c] * r;
                    vv[cl * CPL + c] = a_own[c];
                    const int j = cl * CPL + c;
                    if (j < D) filt[((size_t)sbase + t) * D + j] = a_own[c];
                }
            }
            __syncwarp();
            if (act) {
                rprod *= r;
                const uint32_t bits = __float_as_uint(rprod);
                rexp += (int)((bits >> 23) & 0xffu) - 127;
                rprod = __uint_as_float((bits & 0x807fffffu) | 0x3f800000u);
            }
        }
        if (n > 0 && cl == 0) {
            float s = 0.0f;
            for (int j = 0; j < DP; j++) s += vv[j];
            part = log((double)s) - log((double)rprod) - (double)rexp * (double)kLn2 + msum;
        }
        __syncwarp();
        // ---------------- backward pass + Eq. 14 (lane owns CPL rows; A rows in regs)
        float Arow[CPL][DP];
#pragma unroll
        for (int c = 0; c < CPL; c++)
#pragma unroll
            for (int j = 0; j < DP; j++) Arow[c][j] = lg_A(p, b, cl * CPL + c, j, false);
        float bt[CPL];
#pragma unroll
        for (int c = 0; c < CPL; c++) bt[c] = lsuf[lidx * DP + cl * CPL + c];
        // filtered row of step i and log-likelihood row of step i loaded one iteration ahead
        auto ld_f = [&](int i, float* a) {
#pragma unroll
            for (int c = 0; c < CPL; c++) {
                const int j = cl * CPL + c;
                a[c] = (i >= 0 && i < n && j < D) ? filt[((size_t)sbase + t0 + i) * D + j] : 0.0f;
            }
        };
        float fnext[CPL], lnext[CPL];
        ld_f(nmax - 1, fnext);
        ld_ll(nmax - 1, lnext);
        for (int i = nmax - 1; i >= 0; i--) {
            const bool act = i < n;
            const int64_t t = t0 + i;
            float g[CPL], fa[CPL], lv[CPL];
#pragma unroll
            for (int c = 0; c < CPL; c++) {
                fa[c] = fnext[c];
                lv[c] = lnext[c];
            }
            ld_f(i - 1, fnext);
            if (i > 0) ld_ll(i - 1, lnext);
            float z = 0.0f;
#pragma unroll
            for (int c = 0; c < CPL; c++) {
                g[c] = fa[c] * bt[c];
                z += g[c];
            }
            z = grp_sum<LPL>(z);
            const float rz = rcp(z);
#pragma unroll
            for (int c = 0; c < CPL; c++) {
                const int j = cl * CPL + c;
                if (act && j < D) p.smoothed[((size_t)sbase + t) * D + j] = g[c] * rz;
            }
            if (i > 0) {
                float v[CPL];
#pragma unroll
                for (int c = 0; c < CPL; c++) v[c] = lv[c];
                float m = v[0];
#pragma unroll
                for (int c = 1; c < CPL; c++) m = fmaxf(m, v[c]);
                m = grp_max<LPL>(m);
                if (!(m > neg_inf())) m = 0.0f;
                __syncwarp();
                if (act) {
#pragma unroll
                    for (int c = 0; c < CPL; c++) vv[cl * CPL + c] = ex2((v[c] - m) * kLog2e) * bt[c];
                }
                __syncwarp();
                float y[CPL], q[CPL][4];
#pragma unroll
                for (int c = 0; c < CPL; c++) q[c][0] = q[c][1] = q[c][2] = q[c][3] = 0.0f;
#pragma unroll
                for (int k4 = 0; k4 < DP; k4 += 4) {
                    const float4 x = *reinterpret_cast<const float4*>(vv + k4);
#pragma unroll
                    for (int c = 0; c < CPL; c++) {
                        q[c][0] = fmaf(Arow[c][k4], x.x, q[c][0]);
                        q[c][1] = fmaf(Arow[c][k4 + 1], x.y, q[c][1]);
                        q[c][2] = fmaf(Arow[c][k4 + 2], x.z, q[c][2]);
                        q[c][3] = fmaf(Arow[c][k4 + 3], x.w, q[c][3]);
                    }
                }
#pragma unroll
                for (int c = 0; c < CPL; c++) y[c] = (q[c][0] + q[c][1]) + (q[c][2] + q[c][3]);
                float mx = y[0];
#pragma unroll
                for (int c = 1; c < CPL; c++) mx = fmaxf(mx, y[c]);
                mx = grp_max<LPL>(mx);
                const float sc = pow2_inv(mx);
                if (act) {
#pragma unroll
                    for (int c = 0; c < CPL; c++) bt[c] = y[c] * sc;
                }
            }
        }
    } else {
        // ---------------- Viterbi forward sweep with backpointers (lane owns CPL columns)
        float LAc[CPL][DP], lpv[CPL];
#pragma unroll
        for (int c = 0; c < CPL; c++) {
#pragma unroll
            for (int k = 0; k < DP; k++) LAc[c][k] = lg_A(p, b, k, cl * CPL + c, true);
            lpv[c] = lg_pi(p, b, cl * CPL + c, true);
        }
        uint8_t* og = orig + lidx * DP;
#pragma unroll
        for (int c = 0; c < CPL; c++) {
            vv[cl * CPL + c] = lpre[lidx * DP + cl * CPL + c];
            og[cl * CPL + c] = (uint8_t)(cl * CPL + c);
        }
        __syncwarp();
        double acc = 0.0;
        float V[CPL];
#pragma unroll
        for (int c = 0; c < CPL; c++) V[c] = vv[cl * CPL + c];
        auto ld_llv = [&](int i, float* v) {  // row of step i, loaded one step ahead (as the smoother)
#pragma unroll
            for (int c = 0; c < CPL; c++) {
                const int j = cl * CPL + c;
                v[c] = (i >= 0 && i < n && j < D) ? __ldg(ll + (t0 + i) * D + j) : neg_inf();
            }
        };
        float vnext[CPL];
        ld_llv(0, vnext);
        for (int i = 0; i < nmax; i++) {
            const bool act = i < n;
            const int64_t t = t0 + i;
            float v[CPL];
#pragma unroll
            for (int c = 0; c < CPL; c++) v[c] = vnext[c];
            ld_llv(i + 1, vnext);
            float m = v[0];
#pragma unroll
            for (int c = 1; c < CPL; c++) m = fmaxf(m, v[c]);
            m = grp_max<LPL>(m);
            if (!(m > neg_inf())) m = 0.0f;
            float best[CPL];
            int arg[CPL];
#pragma unroll
            for (int c = 0; c < CPL; c++) {
                best[c] = neg_inf();
                arg[c] = 0;
            }
            if constexpr (CPL == 1) {
                // scores from 16-B broadcast reads, the max by a FMNMX3 tree, then the smallest
                // index attaining it (reading 5) by independent compares: no serial
                // compare-select chain through the DP candidates
                float sc[DP];
#pragma unroll
                for (int k4 = 0; k4 < DP; k4 += 4) {
                    const float4 x = *reinterpret_cast<const float4*>(vv + k4);
                    sc[k4] = x.x +  ((p.t_base + t == 0) ? lpv[0] : LAc[0][k4]);
                    sc[k4 + 1] = x.y +  ((p.t_base + t == 0) ? lpv[0] : LAc[0][k4 + 1]);
                    sc[k4 + 2] = x.z +  ((p.t_base + t == 0) ? lpv[0] : LAc[0][k4 + 2]);
                    sc[k4 + 3] = x.w +  ((p.t_base + t == 0) ? lpv[0] : LAc[0][k4 + 3]);
                }
                const float bm = vmax_tree<DP>(sc);
                int a = 0;
#pragma unroll
                for (int k = DP - 1; k >= 0; k--) a = (sc[k] == bm) ? k : a;
                if (bm > neg_inf()) {
                    best[0] = bm;
                    arg[0] = a;
                }
            } else {
#pragma unroll
                for (int k = 0; k < DP; k++) {
                    const float vk = vv[k];
#pragma unroll
                    for (int c = 0; c < CPL; c++) {
                        const float sc = vk + ((p.t_base + t == 0) ? lpv[c] : LAc[c][k]);
                        if (sc > best[c]) {
                            best[c] = sc;
                            arg[c] = k;
                        }
                    }
                }
            }
            float o = neg_inf(), Vn[CPL];
#pragma unroll
            for (int c = 0; c < CPL; c++) {
                Vn[c] = best[c] + (v[c] - m);
                o = fmaxf(o, Vn[c]);
            }
            o = grp_max<LPL>(o);
            if (!(o > neg_inf())) {
                if (act && p.t_base + t < zero_t) zero_t = p.t_base + t;
                o = 0.0f;
            }
            if (act && cl == 0) acc += (double)(o + m);
            uint8_t on[CPL];
#pragma unroll
            for (int c = 0; c < CPL; c++) on[c] = og[arg[c]];
            __syncwarp();
            if (act) {  // inactive half-warp leaves keep their final V / origin map
#pragma unroll
                for (int c = 0; c < CPL; c++) {
                    const int j = cl * CPL + c;
                    V[c] = Vn[c] - o;
                    vv[j] = V[c];
                    og[j] = on[c];
                    p.bp[((size_t)b * p.T + t) * DP + j] = (uint8_t)arg[c];
                }
            }
            __syncwarp();
        }
        part = acc;
        {
            // x*_{T-1} = smallest argmax of V (reduction warp-uniform, used by the leaf ending at T)
            int xs = DP;
#pragma unroll
            for (int c = CPL - 1; c >= 0; c--)
                if (V[c] == 0.0f && cl * CPL + c < D) xs = cl * CPL + c;
#pragma unroll
            for (int o = 1; o < LPL; o <<= 1) xs = min(xs, __shfl_xor_sync(0xffffffffu, xs, o));
            if (n > 0) {
                // leaf map f(x_end) = state before the leaf
#pragma unroll
                for (int c = 0; c < CPL; c++)
                    p.lmap[((size_t)b * p.NL + L) * DP + cl * CPL + c] = og[cl * CPL + c];
                if (t0 + n == T && cl == 0) p.xstar[b] = xs;
            } else if (L < p.NL) {  // empty leaf (varlen batch): identity map
#pragma unroll
                for (int c = 0; c < CPL; c++)
                    p.lmap[((size_t)b * p.NL + L) * DP + cl * CPL + c] = (uint8_t)(cl * CPL + c);
            }
        }
        __syncthreads();
        // block map = f_first o ... o f_last over this block's leaves (thread x < DP computes entry x)
        if (threadIdx.x < DP) {
            int x = threadIdx.x;
            for (int q = nleaf - 1; q >= 0; q--) x = og_global_lookup(p, b, (int64_t)blk * NLB + q, x, DP);
            p.bmap[((size_t)b * p.NB + blk) * DP + threadIdx.x] = (uint8_t)x;
        }
    }
    // per-leaf partial sums (fixed order later) and info
    if (L < p.NL && cl == 0) p.partial[(size_t)b * p.NL + L] = part;
    if (zero_t != INT64_MAX) atomicMax(zero_code, (1ull << 62) - (unsigned long long)zero_t);
}

// ------------------------------------------------------------------------------------------- K4/K5
__global__ void lg_resolve_kernel(const LgParams p, int DP) {
    // one CTA per sequence: end state of every block = (F_{blk+1} o ... o F_{NB-1})(x*).  The block maps
    // are staged in SMEM (coalesced, chunks of up to 32 KB from the end), so the serial composition runs
    // on SMEM latency instead of one dependent global load per block.
    __shared__ uint8_t smaps[32768];
    __shared__ int xs;
    const int64_t b = blockIdx.x;
    const uint8_t* src = p.bmap + (size_t)b * p.NB * DP;
    const int64_t cb = 32768 / DP;  // blocks per chunk
    if (threadIdx.x == 0) {
        int x = p.xstar[b];
        xs = (x < 0 || x >= DP) ? 0 : x;
    }
    for (int64_t hi = p.NB; hi > 0; hi -= cb) {
        const int64_t lo = hi - cb > 0 ? hi - cb : 0;
        __syncthreads();
        for (int64_t q = threadIdx.x; q < (hi - lo) * DP; q += blockDim.x) smaps[q] = src[lo * DP + q];
        __syncthreads();
        if (threadIdx.x == 0) {
            int x = xs;
            for (int64_t blk = hi - 1; blk >= lo; blk--) {
                p.bend[b * p.NB + blk] = x;
                x = smaps[(blk - lo) * DP + x];
            }
            xs = x;
        }
    }
}

template <int DP>
__global__ void __launch_bounds__(256) lg_backtrack_kernel(const LgParams p) {
    // one thread per leaf backtracks through its backpointers (Alg. 4 lines 8-10) from the leaf's end
    // state; the block's backpointer rows are staged in SMEM in chunks of 32 KB (from the end of the
    // block's range), so each step of the serial walk is an SMEM load, not a dependent global one.
    using C = LG<DP>;
    constexpr int NLB = C::NLB;
    constexpr int CHS = 32768 / DP;  // steps per chunk
    __shared__ int ends[NLB];
    __shared__ __align__(16) uint8_t sbp[CHS * DP];
    const int64_t b = blockIdx.y;
    const int blk = blockIdx.x;
    int64_t sbase, T_raw;  // packed first row / length of sequence b (varlen batches, f4)
    const int64_t T = seq_span(p.offsets, p.T, b, sbase, T_raw);
    int nleaf = NLB;
    if ((int64_t)blk * NLB + nleaf > p.NL) nleaf = (int)(p.NL - (int64_t)blk * NLB);
    if (threadIdx.x == 0) {
        int x = p.bend[b * p.NB + blk];
        for (int q = nleaf - 1; q >= 0; q--) {
            ends[q] = x;
            x = p.lmap[((size_t)b * p.NL + (int64_t)blk * NLB + q) * DP + x];
        }
    }
    __syncthreads();
    const int q = threadIdx.x;
    const int64_t la = ((int64_t)blk * NLB + q) * p.SL;                      // this thread's leaf
    const int64_t lb = (q < nleaf) ? ((la + p.SL < T) ? la + p.SL : T) : la;
    int x = (q < nleaf) ? ends[q] : 0;
    const int64_t r0 = (int64_t)blk * NLB * p.SL;                             // the block's steps
    int64_t r1 = r0 + (int64_t)nleaf * p.SL;
    if (r1 > T) r1 = T;
    const uint8_t* bpg = p.bp + (size_t)b * p.T * DP;
    for (int64_t c1 = r1; c1 > r0; c1 -= CHS) {
        const int64_t c0 = (c1 - CHS > r0) ? c1 - CHS : r0;
        __syncthreads();
        const uint32_t* src = reinterpret_cast<const uint32_t*>(bpg + c0 * DP);
        uint32_t* dst = reinterpret_cast<uint32_t*>(sbp);
        for (int64_t w = threadIdx.x; w < (c1 - c0) * DP / 4; w += blockDim.x) dst[w] = src[w];
        __syncthreads();
        const int64_t hi = (lb < c1) ? lb : c1, lo = (la > c0) ? la : c0;
        for (int64_t t = hi - 1; t >= lo; t--) {
            p.path[(size_t)sbase + t] = x;
            x = sbp[(t - c0) * DP + x];
        }
    }
}

__global__ void lg_finalize_kernel(const LgParams p) {
    // one CTA (256 threads) per sequence: fixed-order sum of the NL partials, info, reset sync words
    __shared__ double red[8];
    const int64_t b = blockIdx.x;
    const int64_t per = (p.NL + 255) / 256;
    double v = 0.0;
    for (int64_t i = threadIdx.x * per; i < (threadIdx.x + 1) * per && i < p.NL; i++) v += p.partial[b * p.NL + i];
#pragma unroll
    for (int st = 16; st >= 1; st >>= 1) v += __shfl_down_sync(0xffffffffu, v, st);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < 8; w++) s += red[w];
        p.scalar_out[b] = s;
        uint32_t* sync = reinterpret_cast<uint32_t*>(p.ws_sync + b * 64);
        unsigned long long* zero_code = reinterpret_cast<unsigned long long*>(sync + 4);
        const uint32_t badf = atomicExch(sync + 8, 0u);
        const unsigned long long zc = atomicExch(zero_code, 0ull);
        int32_t inf = 0;
        if (badf) inf = -1;
        else if (zc) inf = (int32_t)((1ull << 62) - zc + 1ull);
        int64_t sb, raw;
        seq_span(p.offsets, p.T, b, sb, raw);
        if (raw < 1 || raw > p.T) inf = kInfoBadLength;
        p.info[b] = inf;
    }
}

// ------------------------------------------------------------------------------------------- host
// Split phase: the carries entering and leaving this rank's slice from the gathered rank aggregates
// (one CTA, DP threads): forward = 1^T Agg_0 ... Agg_{rank-1}, backward = Agg_{rank+1} ... Agg_{W-1} 1,
// each step renormalised by an exact power of two (Thms 1-2 across ranks).
// Split-phase Viterbi (max-product): the forward carry entering this rank, 0 (x) Agg_0 ... Agg_{rank-1}
// in the max-plus semiring (Prop. 2 across ranks), normalised to max 0.
template <int DP>
__global__ void __launch_bounds__(DP) lg_rank_carry_mp_kernel(const LgParams p) {
    __shared__ float u[DP], red[DP];
    const int j = threadIdx.x;
    u[j] = 0.0f;
    __syncthreads();
    for (int q = 0; q < p.rank; q++) {
        const float* M = p.agg_all + (size_t)q * DP * DP;
        float y = neg_inf();
        for (int k = 0; k < DP; k++) y = fmaxf(y, u[k] + __ldg(M + k * DP + j));
        red[j] = y;
        __syncthreads();
        float m = neg_inf();
        for (int k = 0; k < DP; k++) m = fmaxf(m, red[k]);
        __syncthreads();
        u[j] = (m > neg_inf()) ? y - m : y;
        __syncthreads();
    }
    p.rcar[j] = u[j];
}
// Viterbi forward (split phase): this rank's record = the composition of its block maps, F(x) = the
// state before the rank's first step reached by backtracking from x at its last step, and x* = the
// smallest argmax of V at its last step (used when this rank ends the sequence).
__global__ void lg_rank_record_kernel(const LgParams p, int DP) {
    const int x0 = threadIdx.x;
    if (x0 < DP) {
        int x = x0;
        for (int64_t blk = p.NB - 1; blk >= 0; blk--) x = p.bmap[(size_t)blk * DP + x];
        p.rec_out[x0] = (uint8_t)x;
    }
    if (x0 == 0) *reinterpret_cast<int32_t*>(p.rec_out + DP) = p.xstar[0];
}
// Viterbi finish (split phase): this rank's end state from the gathered records: x* of the last rank
// mapped back through the ranks to our right; it seeds the block resolve.  Finish only backtracks:
// info = 0 (errors were reported by reduce / forward).
__global__ void lg_rank_end_kernel(const LgParams p, int DP) {
    if (threadIdx.x != 0) return;
    int x = *reinterpret_cast<const int32_t*>(p.rec_all + (size_t)(p.world - 1) * p.rec_bytes + DP);
    for (int q = p.world - 1; q > p.rank; q--) x = p.rec_all[(size_t)q * p.rec_bytes + (x < 0 ? 0 : x)];
    p.xstar[0] = x;
    p.info[0] = 0;
}

template <int DP>
__global__ void __launch_bounds__(DP) lg_rank_carry_kernel(const LgParams p) {
    __shared__ float u[DP], w[DP];
    __shared__ float red[DP];
    const int j = threadIdx.x;
    u[j] = 1.0f;
    w[j] = 1.0f;
    __syncthreads();
    auto renorm = [&](float y, float* dst) {
        red[j] = y;
        __syncthreads();
        float m = 0.0f;
        for (int k = 0; k < DP; k++) m = fmaxf(m, red[k]);
        __syncthreads();
        dst[j] = y * pow2_inv(m);
        __syncthreads();
    };
    for (int q = 0; q < p.rank; q++) {  // u <- u Agg_q
        const float* M = p.agg_all + (size_t)q * DP * DP;
        float y = 0.0f;
        for (int k = 0; k < DP; k++) y = fmaf(u[k], __ldg(M + k * DP + j), y);
        renorm(y, u);
    }
    for (int q = p.world - 1; q > p.rank; q--) {  // w <- Agg_q w
        const float* M = p.agg_all + (size_t)q * DP * DP;
        float y = 0.0f;
        for (int k = 0; k < DP; k++) y = fmaf(__ldg(M + j * DP + k), w[k], y);
        renorm(y, w);
    }
    p.rcar[j] = u[j];
    p.rcar[DP + j] = w[j];
}
// Split-phase reduce: input errors (NaN / +inf seen by the leaf kernels) -> info, flag cleared.
__global__ void lg_reduce_info_kernel(const LgParams p) {
    uint32_t* bad = reinterpret_cast<uint32_t*>(p.ws_sync) + 8;
    const uint32_t f = atomicExch(bad, 0u);
    p.info[0] = f ? -1 : 0;
}

template <int DP, int OP>
static cudaError_t lg_launch(const LgParams& p, cudaStream_t s) {
    using C = LG<DP>;
    const size_t sm1 = (size_t)C::NLB * DP * DP * 4;
    if (cudaError_t e = ensure_smem_optin(reinterpret_cast<const void*>(lg_leaf_kernel<DP, OP>), sm1); e != cudaSuccess)
        return e;
    const size_t sm3 = (size_t)(3 * C::NLB + 2) * DP * 4 + (size_t)C::NLB * DP + 64;
    if (cudaError_t e = ensure_smem_optin(reinterpret_cast<const void*>(lg_sweep_kernel<DP, OP>), sm3); e != cudaSuccess)
        return e;
    const dim3 grid((unsigned)p.NB, (unsigned)p.B);
    const size_t smg = (size_t)3 * DP * DP * 4;
    if (cudaError_t e = ensure_smem_optin(reinterpret_cast<const void*>(lg_group_kernel<DP, OP>), smg); e != cudaSuccess)
        return e;
    const bool do_leaf = (p.mode == HMM_MODE_FULL || p.mode == HMM_MODE_REDUCE);
    if (do_leaf) {
        if (OP == 0 && DP == 64 && p.tc) {
            cudaError_t e = launch_large_tc_leaf(p, p.lik, s);
            if (e != cudaSuccess) return e;
        }
        lg_leaf_kernel<DP, OP><<<grid, 256, sm1, s>>>(p);
        if (p.NG > 1)  // group products (also the first level of the rank aggregate)
            lg_group_kernel<DP, OP><<<dim3((unsigned)p.NG, (unsigned)p.B), 256, smg, s>>>(p, p.groot, p.NB, p.KG, p.NG,
                                                                                          p.gprod);
    }
    if (p.mode == HMM_MODE_REDUCE) {  // the rank aggregate = the ordered product of every block root
        if (p.NG > 1) lg_group_kernel<DP, OP><<<dim3(1, 1), 256, smg, s>>>(p, p.gprod, p.NG, p.NG, 1, p.agg_out);
        else lg_group_kernel<DP, OP><<<dim3(1, 1), 256, smg, s>>>(p, p.groot, p.NB, p.NB, 1, p.agg_out);
        lg_reduce_info_kernel<<<1, 1, 0, s>>>(p);
        return cudaGetLastError();
    }
    if (p.mode == HMM_MODE_VFINISH) {  // backtrack only, from the end state the records give
        lg_rank_end_kernel<<<1, 32, 0, s>>>(p, DP);
        lg_resolve_kernel<<<(unsigned)p.B, 256, 0, s>>>(p, DP);
        lg_backtrack_kernel<DP><<<grid, 256, 0, s>>>(p);
        return cudaGetLastError();
    }
    const float* init_pre = nullptr;
    const float* init_suf = nullptr;
    if (p.mode == HMM_MODE_SFINISH) {
        lg_rank_carry_kernel<DP><<<1, DP, 0, s>>>(p);
        init_pre = p.rcar;
        init_suf = p.rcar + DP;
    } else if (p.mode == HMM_MODE_VFORWARD) {
        lg_rank_carry_mp_kernel<DP><<<1, DP, 0, s>>>(p);
        init_pre = p.rcar;
    }
    {
        const size_t smc = (size_t)6 * DP * DP * 4;
        if (cudaError_t e = ensure_smem_optin(reinterpret_cast<const void*>(lg_carry_kernel<DP, OP>), smc);
            e != cudaSuccess)
            return e;
        if (p.NG <= 1) {  // one level: the chain over the NB block roots
            const LgChain ch{p.groot, p.NB, p.NB * DP * DP, p.NB, 1, init_pre, init_suf, p.bpre, p.bsuf};
            lg_carry_kernel<DP, OP><<<dim3((unsigned)p.B, 2), 64, smc, s>>>(p, ch);
        } else {  // two levels: the chain over the group products, then the chains inside the groups
            const LgChain top{p.gprod, p.NG, p.NG * DP * DP, p.NG, 1, init_pre, init_suf, p.gpre, p.gsuf};
            lg_carry_kernel<DP, OP><<<dim3((unsigned)p.B, 2), 64, smc, s>>>(p, top);
            const LgChain low{p.groot, p.NB, p.NB * DP * DP, p.KG, p.NG, p.gpre, p.gsuf, p.bpre, p.bsuf};
            lg_carry_kernel<DP, OP><<<dim3((unsigned)(p.B * p.NG), 2), 64, smc, s>>>(p, low);
        }
    }
    lg_sweep_kernel<DP, OP><<<grid, 256, sm3, s>>>(p);
    if (OP == 1 && p.mode == HMM_MODE_FULL) {
        lg_resolve_kernel<<<(unsigned)p.B, 256, 0, s>>>(p, DP);
        lg_backtrack_kernel<DP><<<grid, 256, 0, s>>>(p);
    }
    lg_finalize_kernel<<<(unsigned)p.B, 256, 0, s>>>(p);
    if (OP == 1 && p.mode == HMM_MODE_VFORWARD) lg_rank_record_kernel<<<1, 64, 0, s>>>(p, DP);
    return cudaGetLastError();
}

cudaError_t launch_large(int DP, int op, const LgParams& p, cudaStream_t s) {
    switch (DP) {
        case 16: return op == 0 ? lg_launch<16, 0>(p, s) : lg_launch<16, 1>(p, s);
        case 32: return op == 0 ? lg_launch<32, 0>(p, s) : lg_launch<32, 1>(p, s);
        case 64: return op == 0 ? lg_launch<64, 0>(p, s) : lg_launch<64, 1>(p, s);
        default: return cudaErrorInvalidValue;
    }
}

int large_leaves_per_block(int DP) { return DP == 16 ? LG<16>::NLB : (DP == 32 ? LG<32>::NLB : LG<64>::NLB); }

}  // namespace hmm
