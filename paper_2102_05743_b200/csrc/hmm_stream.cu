// hmm_stream.cu — lane-streaming parallel scan for long single sequences, 1 <= D <= 8, sm_100a.
//
// Same method as hmm_small.cu (Algorithm 3 / Algorithm 5 with block-wise elements, PAPER.md:408-426,
// 722-740, 759-760), decomposed for sequences too long to stay resident in shared memory:
//
//   lane   thread g = c*NT + tid of CTA c owns the contiguous steps [g*n, min((g+1)*n, T)) and walks
//          them in slices of S steps staged in a private SMEM slot of a 3-deep ring; a warp moves its
//          32 lane slices cooperatively (cp.async 16 B per thread, coalesced), so loads run two
//          slices ahead of the math without any CTA-wide synchronisation inside the passes.
//   pass 1 each lane folds its range right-to-left into one D x D aggregate (Def. 3 matrix product /
//          Def. 5 max-plus product).  The smoother also stores, per slice k, the product Q_k of the
//          lane's slices right of k (the suffix that turns the lane's backward carry into the
//          backward potential at the end of slice k, Thm. 2), so pass 2 needs no second fold.
//   scan   lane aggregates -> CTA tree (SMEM) -> grid exchange of the G CTA roots (global memory,
//          arrival counter, cooperative launch) -> lane carries: forward potential a_{0:k} (Thm. 1),
//          backward potential (Thm. 2), or the max-product forward carry (Alg. 5).
//   pass 2 smoother: per slice, the forward filter continues the lane's running alpha (Alg. 1 forward,
//          normalised; log Z by telescoping the applied multipliers over the whole lane), the
//          backward pass starts from Q_k times the lane's backward carry, Eq. 14 gives the smoothed
//          marginals; both outputs leave by warp-cooperative streaming stores.  Viterbi: forward sweep with
//          backpointers (Alg. 4 lines 3-6) written to the workspace, lane backpointer map composed.
//   pass 3 Viterbi: lane end states from the map tree / exchange, backtrack slice by slice.
//
// Pass 1 runs right-to-left so that the slices it loads last (the first slice of every lane) are the
// first pass 2 reads: up to ~L2-size of the re-read is served from the 126 MB L2.
#include <cstdint>
#include <cstring>

#include "hmm_device.cuh"
#include "hmm_plan.h"
#include "hmm_small_ops.cuh"

#ifndef HMM_SP_TWO_CHAIN
#define HMM_SP_TWO_CHAIN 1
#endif

namespace hmm {

// ---------------------------------------------------------------------------- slice folds
// Where step i of a slice reads its log-likelihood row: the staged rows, or (symbol inputs, SURVEY.md
// §8(f) f1) the emission table row of the staged symbol, log_B[:, y_i] (Eq. 5b).
template <int D, bool SY>
struct RowSrc {
    const float* rows;
    const uint8_t* ys;
    const float* tab;
    __device__ __forceinline__ const float* operator()(int i) const {
        if constexpr (SY) return tab + (int)ys[i] * D;
        else return rows + i * D;
    }
};
// Sum-product, right to left over one slice: P <- psi_t P for t = nr-1 .. 0 (psi_t = A diag(l_t),
// psi_0 = 1 (pi o l_0)^T when the slice starts the sequence).  Renormalisation is exact and free: the
// power-of-two factor 2^d that brings max(P) into [1,2) is added to the next step's ex2 argument,
// l_t = 2^(log2e (ll_t - m_t) + d), so a step costs D^3 FMA + D^2 FMUL (A diag(l)) + D FFMA + D MUFU +
// the max tree.  `d` carries the pending offset between slices.  An impossible step (all -inf) gives
// l = 0; NaN / +inf inputs turn into NaN through ll - m and are caught by the caller's final check.
template <int D>
__device__ __forceinline__ void sp_back_step(const float* row, bool t0, const float* A, const float* pi, float* P,
                                             float& d) {
    float v[D], l[D];
    ld_row<D>(row, v);
    const float m = fmaxf(vmax2_tree<D>(v), -1e30f);  // all -inf (impossible step): l = 0, -m*log2e stays finite
    const float c = fmaf(-m, kLog2e, d);
#pragma unroll
    for (int j = 0; j < D; j++) l[j] = ex2(fmaf(v[j], kLog2e, c));
    float Pn[D * D];
    if (t0) {
        float r[D];
#pragma unroll
        for (int j = 0; j < D; j++) {
            float acc = (pi[0] * l[0]) * P[j];
#pragma unroll
            for (int k = 1; k < D; k++) acc = fmaf(pi[k] * l[k], P[k * D + j], acc);
            r[j] = acc;
        }
#pragma unroll
        for (int i = 0; i < D; i++)
#pragma unroll
            for (int j = 0; j < D; j++) Pn[i * D + j] = r[j];
    } else {
#pragma unroll
        for (int i = 0; i < D; i++) {
            float a[D];
#pragma unroll
            for (int k = 0; k < D; k++) a[k] = A[i * D + k] * l[k];
#pragma unroll
            for (int j = 0; j < D; j++) {
                float acc = a[0] * P[j];
#pragma unroll
                for (int k = 1; k < D; k++) acc = fmaf(a[k], P[k * D + j], acc);
                Pn[i * D + j] = acc;
            }
        }
    }
#pragma unroll
    for (int e = 0; e < D * D; e++) P[e] = Pn[e];
    d = exp_offset(vmax2_tree<D * D>(P));
}
// The same step (t > 0, even D) on packed pairs: P2[k*H + jj] = (P(k,2jj), P(k,2jj+1)), H = D/2, and
// A2[i*D + k] = (A(i,k), A(i,k)).  psi_t P = A (diag(l_t) P): diag(l) P is D*H FMUL2, the product D*D*H
// FFMA2/FMUL2 -- the same D^3 + D^2 FP32 multiply-adds as the scalar step (bit-identical roundings
// per element are not needed: only the operand order differs), in half the issue slots.  The fold is
// issue-bound, so the freed slots absorb the MUFU/FMNMX/integer work.
template <int D>
__device__ __forceinline__ void sp_back_step2(const float* row, const float2* A2, float2* P2, float& d) {
    constexpr int H = D / 2;
    float v[D];
    ld_row<D>(row, v);
    const float m = fmaxf(vmax2_tree<D>(v), -1e30f);
    const float c = fmaf(-m, kLog2e, d);
    float2 R[D * H];
#pragma unroll
    for (int k = 0; k < D; k++) {
        const float lk = ex2(fmaf(v[k], kLog2e, c));
        const float2 l2 = make_float2(lk, lk);
#pragma unroll
        for (int jj = 0; jj < H; jj++) R[k * H + jj] = __fmul2_rn(l2, P2[k * H + jj]);
    }
#pragma unroll
    for (int i = 0; i < D; i++) {
#pragma unroll
        for (int jj = 0; jj < H; jj++) {
            float2 acc = __fmul2_rn(A2[i * D], R[jj]);
#pragma unroll
            for (int k = 1; k < D; k++) acc = __ffma2_rn(A2[i * D + k], R[k * H + jj], acc);
            P2[i * H + jj] = acc;
        }
    }
    float mx[D * H];
#pragma unroll
    for (int e = 0; e < D * H; e++) mx[e] = fmaxf(P2[e].x, P2[e].y);
    d = exp_offset(vmax2_tree<D * H>(mx));
}
// Start of a chain: X = psi_t = A diag(l_t) (packed pairs as in sp_back_step2), d = its offset.
template <int D>
__device__ __forceinline__ void sp_chain_start2(const float* row, const float2* A2, float2* X2, float& d) {
    constexpr int H = D / 2;
    float v[D];
    ld_row<D>(row, v);
    const float m = fmaxf(vmax2_tree<D>(v), -1e30f);
    const float c = -m * kLog2e;
    float l[D];
#pragma unroll
    for (int k = 0; k < D; k++) l[k] = ex2(fmaf(v[k], kLog2e, c));
#pragma unroll
    for (int i = 0; i < D; i++)
#pragma unroll
        for (int jj = 0; jj < H; jj++) X2[i * H + jj] = __fmul2_rn(make_float2(A2[i * D + 2 * jj].x, A2[i * D + 2 * jj + 1].x),
                                                    make_float2(l[2 * jj], l[2 * jj + 1]));
    float mx[D * H];
#pragma unroll
    for (int e = 0; e < D * H; e++) mx[e] = fmaxf(X2[e].x, X2[e].y);
    d = exp_offset(vmax2_tree<D * H>(mx));
}
// One slice, right to left (sum-product).  D = 2, 4 run the packed-pair steps; full slices that do not
// start the sequence are folded as two chains (as the max-product fold below): with the packed step the
// issue slots are no longer the limit, and the 2x ILP took the T=1e8 smoother from 1.36 to 1.32 ms
// (with scalar steps the fold was issue-bound and the combine only added work).  Other slices, and
// odd D / D > 4, keep one chain.  HMM_SP_TWO_CHAIN=0 builds the one-chain packed fold for comparison.
template <int D, int S, class RS>
__device__ __forceinline__ void sp_fold_back(const RS rows, int nr, bool t0, const float* A, const float* pi,
                                             float* P, float& d) {
    if constexpr (D % 2 == 0 && D <= 4) {  // (D = 6, 8: the packed operands would spill)
        constexpr int H = D / 2;
        float2 A2[D * D], P2[D * H];
#pragma unroll
        for (int e = 0; e < D * D; e++) A2[e] = make_float2(A[e], A[e]);
#if HMM_SP_TWO_CHAIN
        if (nr == S && !t0) {
            // two independent chains X = psi_{S/2} .. psi_{S-1}, Y = psi_0 .. psi_{S/2-1} (2x ILP for
            // the latency-bound step chain), combined as P <- Y (X P); each chain starts from psi itself,
            // which saves exactly the products the combine costs.  Scales are free (pass 1 keeps only
            // normalised products).
            constexpr int HS = S / 2;
            float2 X2[D * H], Y2[D * H];
            float dx = 0.0f, dy = 0.0f;
            sp_chain_start2<D>(rows(S - 1), A2, X2, dx);
            sp_chain_start2<D>(rows(HS - 1), A2, Y2, dy);
#pragma unroll 2
            for (int q = 1; q < HS; q++) {
                sp_back_step2<D>(rows(S - 1 - q), A2, X2, dx);
                sp_back_step2<D>(rows(HS - 1 - q), A2, Y2, dy);
            }
            float X[D * D], Y[D * D], XP[D * D];
#pragma unroll
            for (int e = 0; e < D * H; e++) {
                X[2 * e] = X2[e].x;
                X[2 * e + 1] = X2[e].y;
                Y[2 * e] = Y2[e].x;
                Y[2 * e + 1] = Y2[e].y;
            }
            mat_op<D, false>(X, P, XP);
            mat_op<D, false>(Y, XP, P);
            d = 0.0f;
            return;
        }
#endif
#pragma unroll
        for (int e = 0; e < D * H; e++) P2[e] = make_float2(P[2 * e], P[2 * e + 1]);
        if (nr == S) {
#pragma unroll 4
            for (int ii = S - 1; ii >= 1; ii--) sp_back_step2<D>(rows(ii), A2, P2, d);
        } else {
#pragma unroll 1
            for (int ii = nr - 1; ii >= 1; ii--) sp_back_step2<D>(rows(ii), A2, P2, d);
        }
#pragma unroll
        for (int e = 0; e < D * H; e++) {
            P[2 * e] = P2[e].x;
            P[2 * e + 1] = P2[e].y;
        }
    } else {
        if (nr == S) {
#pragma unroll 4
            for (int ii = S - 1; ii >= 1; ii--) sp_back_step<D>(rows(ii), false, A, pi, P, d);
        } else {
#pragma unroll 1
            for (int ii = nr - 1; ii >= 1; ii--) sp_back_step<D>(rows(ii), false, A, pi, P, d);
        }
    }
    sp_back_step<D>(rows(0), t0, A, pi, P, d);
}

// Max-product (log domain), one step right to left: P(i,j) <- max_k (LA(i,k) + w_t(k) + P(k,j)),
// w_t = ll_t - m_t (row-independent LP(k) + w_0(k) for the sequence's first step).  `chk` collects
// NaN evidence.
template <int D>
__device__ __forceinline__ void mp_back_step(const float* row, bool t0, const float* LA, const float* LP, float* P,
                                             float& chk) {
    float v[D], W[D * D];
    ld_row<D>(row, v);
    float m = vmax<D>(v);
    if (!(m > neg_inf())) m = 0.0f;
    float w[D];
#pragma unroll
    for (int k = 0; k < D; k++) w[k] = v[k] - m;
    chk += vsum<D>(w);
#pragma unroll
    for (int k = 0; k < D; k++)
#pragma unroll
        for (int j = 0; j < D; j++) W[k * D + j] = w[k] + P[k * D + j];
    float Pn[D * D];
#pragma unroll
    for (int i = 0; i < D; i++) {
#pragma unroll
        for (int j = 0; j < D; j++) {
            float sc[D];
#pragma unroll
            for (int k = 0; k < D; k++) sc[k] = (t0 ? LP[k] : LA[i * D + k]) + W[k * D + j];
            Pn[i * D + j] = vmax<D>(sc);
        }
    }
#pragma unroll
    for (int e = 0; e < D * D; e++) P[e] = Pn[e];
}
template <int D>
__device__ __forceinline__ void mp_chain_start(const float* row, const float* LA, float* X, float& chk) {
    float v[D];
    ld_row<D>(row, v);
    float m = vmax<D>(v);
    if (!(m > neg_inf())) m = 0.0f;
    float w[D];
#pragma unroll
    for (int k = 0; k < D; k++) w[k] = v[k] - m;
    chk += vsum<D>(w);
#pragma unroll
    for (int i = 0; i < D; i++)
#pragma unroll
        for (int k = 0; k < D; k++) X[i * D + k] = LA[i * D + k] + w[k];
}
// mp_back_step (t > 0, even D) on packed pairs along j: P2[k*H + jj] = (P(k,2jj), P(k,2jj+1)),
// LA2[i*D + k] = (LA(i,k), LA(i,k)).  The D^2 + D^3 adds run as FADD2 with the same operands and order
// as the scalar step (LA + (w + P)), so the results are bit-identical; the maxima stay scalar.
template <int D>
__device__ __forceinline__ void mp_back_step2(const float* row, const float2* LA2, float2* P2, float& chk) {
    constexpr int H = D / 2;
    float v[D];
    ld_row<D>(row, v);
    float m = vmax<D>(v);
    if (!(m > neg_inf())) m = 0.0f;
    float w[D];
#pragma unroll
    for (int k = 0; k < D; k++) w[k] = v[k] - m;
    chk += vsum<D>(w);
    float2 W2[D * H];
#pragma unroll
    for (int k = 0; k < D; k++) {
        const float2 wk = make_float2(w[k], w[k]);
#pragma unroll
        for (int jj = 0; jj < H; jj++) W2[k * H + jj] = __fadd2_rn(wk, P2[k * H + jj]);
    }
#pragma unroll
    for (int i = 0; i < D; i++) {
#pragma unroll
        for (int jj = 0; jj < H; jj++) {
            float sx[D], sy[D];
#pragma unroll
            for (int k = 0; k < D; k++) {
                const float2 s = __fadd2_rn(LA2[i * D + k], W2[k * H + jj]);
                sx[k] = s.x;
                sy[k] = s.y;
            }
            P2[i * H + jj] = make_float2(vmax<D>(sx), vmax<D>(sy));
        }
    }
}
// Max-product slice fold, two interleaved chains for full slices (as sp_fold_back, Def. 5).
template <int D, int S, class RS>
__device__ __forceinline__ void mp_fold_back(const RS rows, int nr, bool t0, const float* LA, const float* LP,
                                             float* P, float& chk) {
    if constexpr (D % 2 == 0 && D <= 4) {  // (D = 6, 8: the packed operands would spill)
        if (nr == S) {
            constexpr int H = D / 2, HS = S / 2;
            float2 LA2[D * D];
#pragma unroll
            for (int e = 0; e < D * D; e++) LA2[e] = make_float2(LA[e], LA[e]);
            float X[D * D], Y[D * D];
            mp_chain_start<D>(rows(S - 1), LA, X, chk);
            mp_chain_start<D>(rows(HS - 1), LA, Y, chk);
            float2 X2[D * H], Y2[D * H];
#pragma unroll
            for (int e = 0; e < D * H; e++) {
                X2[e] = make_float2(X[2 * e], X[2 * e + 1]);
                Y2[e] = make_float2(Y[2 * e], Y[2 * e + 1]);
            }
#pragma unroll 2
            for (int q = 1; q < HS - 1; q++) {
                mp_back_step2<D>(rows(S - 1 - q), LA2, X2, chk);
                mp_back_step2<D>(rows(HS - 1 - q), LA2, Y2, chk);
            }
            mp_back_step2<D>(rows(HS), LA2, X2, chk);
#pragma unroll
            for (int e = 0; e < D * H; e++) {
                X[2 * e] = X2[e].x;
                X[2 * e + 1] = X2[e].y;
                Y[2 * e] = Y2[e].x;
                Y[2 * e + 1] = Y2[e].y;
            }
            mp_back_step<D>(rows(0), t0, LA, LP, Y, chk);
            float XP[D * D];
            mat_op<D, true>(X, P, XP);
            mat_op<D, true>(Y, XP, P);
            return;
        }
    }
    if (nr == S) {
        constexpr int H = S / 2;
        float X[D * D], Y[D * D];
        mp_chain_start<D>(rows(S - 1), LA, X, chk);
        mp_chain_start<D>(rows(H - 1), LA, Y, chk);
#pragma unroll 2
        for (int q = 1; q < H - 1; q++) {
            mp_back_step<D>(rows(S - 1 - q), false, LA, LP, X, chk);
            mp_back_step<D>(rows(H - 1 - q), false, LA, LP, Y, chk);
        }
        mp_back_step<D>(rows(H), false, LA, LP, X, chk);
        mp_back_step<D>(rows(0), t0, LA, LP, Y, chk);
        float XP[D * D];
        mat_op<D, true>(X, P, XP);
        mat_op<D, true>(Y, XP, P);
    } else {
#pragma unroll 1
        for (int ii = nr - 1; ii >= 0; ii--) mp_back_step<D>(rows(ii), ii == 0 && t0, LA, LP, P, chk);
    }
}

// Forward filter over one slice, continuing the lane's alpha.  The log-Z bookkeeping (running
// product of the applied multipliers with its exponent split off, sum of m_t) persists across the
// lane's slices and is closed once per lane (see sp_alpha in hmm_small_ops.cuh); m_t is summed in
// fp32 within the slice (<= 64 terms) and added to the fp64 total once per slice.  Rows are turned
// into l_t in place; filtered rows go to `frows`.  Returns the first zero-mass row, or -1.
template <int D>
__device__ __forceinline__ bool sp_alpha_step(const float* srow, float* row, float* frow, bool t0, const float* A,
                                              const float* pi, float* alpha, float& rprod, int& rexp, float& msl) {
    float l[D];
    ld_row<D>(srow, l);
    const float m = vmax<D>(l);
    const bool ok = m > -FLT_MAX;  // false: impossible step (all -inf), l = 0
    msl += ok ? m : 0.0f;
    const float c0 = ok ? -m * kLog2e : 0.0f;
#pragma unroll
    for (int j = 0; j < D; j++) l[j] = ex2(fmaf(l[j], kLog2e, c0));
    st_row<D>(row, l);
    float ah[D];
    if (t0) {
#pragma unroll
        for (int j = 0; j < D; j++) ah[j] = pi[j] * l[j];
    } else {
#pragma unroll
        for (int j = 0; j < D; j++) {
            float acc = alpha[0] * A[j];
#pragma unroll
            for (int k = 1; k < D; k++) acc = fmaf(alpha[k], A[k * D + j], acc);
            ah[j] = acc * l[j];
        }
    }
    const float c = vsum<D>(ah);
    const float r = rcp(c);
#pragma unroll
    for (int j = 0; j < D; j++) alpha[j] = ah[j] * r;
    st_row<D>(frow, alpha);
    rprod *= r;
    const uint32_t bits = __float_as_uint(rprod);
    rexp += (int)((bits >> 23) & 0xffu) - 127;
    rprod = __uint_as_float((bits & 0x807fffffu) | 0x3f800000u);
    return c > 0.0f;
}
template <int D, int S, class RS>
__device__ __forceinline__ int sp_alpha_slice(const RS src, float* rows, float* frows, int nr, bool t0, const float* A,
                                              const float* pi, float* alpha, float& rprod, int& rexp,
                                              double& msum) {
    int zero_i = -1;
    float msl = 0.0f;
    if (!sp_alpha_step<D>(src(0), rows, frows, t0, A, pi, alpha, rprod, rexp, msl)) zero_i = 0;
    if (nr == S) {
#pragma unroll 4
        for (int i = 1; i < S; i++)
            if (!sp_alpha_step<D>(src(i), rows + i * D, frows + i * D, false, A, pi, alpha, rprod, rexp, msl) &&
                zero_i < 0)
                zero_i = i;
    } else {
#pragma unroll 1
        for (int i = 1; i < nr; i++)
            if (!sp_alpha_step<D>(src(i), rows + i * D, frows + i * D, false, A, pi, alpha, rprod, rexp, msl) &&
                zero_i < 0)
                zero_i = i;
    }
    msum += (double)msl;
    return zero_i;
}

// Backward pass over one slice from the backward potential at its last step, combined with Eq. 14
// (smoothed_t = alpha_t beta_t / Z_t, written over the l rows).
template <int D>
__device__ __forceinline__ void sp_beta_step(float* lrow, const float* frow, const float* A, float* beta) {
    float l[D], a[D], g[D];
    ld_row<D>(lrow, l);
    ld_row<D>(frow, a);
#pragma unroll
    for (int j = 0; j < D; j++) g[j] = a[j] * beta[j];
    const float z = rcp(vsum<D>(g));
#pragma unroll
    for (int j = 0; j < D; j++) g[j] *= z;
    st_row<D>(lrow, g);
    float w[D], bn[D];
#pragma unroll
    for (int j = 0; j < D; j++) w[j] = l[j] * beta[j];
#pragma unroll
    for (int r = 0; r < D; r++) {
        float acc = A[r * D] * w[0];
#pragma unroll
        for (int j = 1; j < D; j++) acc = fmaf(A[r * D + j], w[j], acc);
        bn[r] = acc;
    }
    const float sc = pow2_inv(vmax<D>(bn));
#pragma unroll
    for (int r = 0; r < D; r++) beta[r] = bn[r] * sc;
}
template <int D, int S>
__device__ __forceinline__ void sp_beta_slice(float* lrows, const float* frows, int nr, const float* A, float* beta) {
    if (nr == S) {
#pragma unroll 4
        for (int i = S - 1; i >= 0; i--) sp_beta_step<D>(lrows + i * D, frows + i * D, A, beta);
    } else {
#pragma unroll 1
        for (int i = nr - 1; i >= 0; i--) sp_beta_step<D>(lrows + i * D, frows + i * D, A, beta);
    }
}

// Backward pass + Eq. 14 as sp_beta_slice, also accumulating the Baum-Welch E-step statistics
// (PAPER.md:762-763): the pairwise posterior xi_t(i,j) = a_{t-1}(i) A(i,j) l_t(j) b_t(j) / z_t with the
// normaliser z_t = a_{t-1} . (A (l_t o b_t)) -- the product the backward update computes anyway --
// and the occupancies gamma_t = smoothed_t.  `aprev` is the filtered row entering the slice;
// `skip0` drops xi at the sequence's first step (no predecessor).  Partials are fp32 per slice.
template <int D>
__device__ __forceinline__ void sp_beta_stats_step(float* lrow, const float* frow, const float* aprev,
                                                   const float* A, float* beta, bool want_xi, float* xi,
                                                   float* gs) {
    float l[D], a[D], g[D];
    ld_row<D>(lrow, l);
    ld_row<D>(frow, a);
#pragma unroll
    for (int j = 0; j < D; j++) g[j] = a[j] * beta[j];
    const float zz = rcp(vsum<D>(g));
#pragma unroll
    for (int j = 0; j < D; j++) {
        g[j] *= zz;
        gs[j] += g[j];
    }
    st_row<D>(lrow, g);
    float w[D], bn[D];
#pragma unroll
    for (int j = 0; j < D; j++) w[j] = l[j] * beta[j];
#pragma unroll
    for (int r = 0; r < D; r++) {
        float acc = A[r * D] * w[0];
#pragma unroll
        for (int j = 1; j < D; j++) acc = fmaf(A[r * D + j], w[j], acc);
        bn[r] = acc;
    }
    if (want_xi) {
        float ap[D];
        ld_row<D>(aprev, ap);
        float z = ap[0] * bn[0];
#pragma unroll
        for (int r = 1; r < D; r++) z = fmaf(ap[r], bn[r], z);
        const float rz = (z > 0.0f) ? 1.0f / z : 0.0f;
#pragma unroll
        for (int r = 0; r < D; r++) {
            const float ar = ap[r] * rz;
#pragma unroll
            for (int j = 0; j < D; j++) xi[r * D + j] = fmaf(ar, A[r * D + j] * w[j], xi[r * D + j]);
        }
    }
    const float sc = pow2_inv(vmax<D>(bn));
#pragma unroll
    for (int r = 0; r < D; r++) beta[r] = bn[r] * sc;
}
template <int D, int S>
__device__ __forceinline__ void sp_beta_slice_stats(float* lrows, const float* frows, int nr, const float* A,
                                                    float* beta, const float* aprev, bool skip0, double* xi_l,
                                                    double* g_l) {
    float xi[D * D], gs[D];
#pragma unroll
    for (int e = 0; e < D * D; e++) xi[e] = 0.0f;
#pragma unroll
    for (int d = 0; d < D; d++) gs[d] = 0.0f;
#pragma unroll 1
    for (int i = nr - 1; i >= 1; i--) sp_beta_stats_step<D>(lrows + i * D, frows + i * D, frows + (i - 1) * D, A, beta, true, xi, gs);
    sp_beta_stats_step<D>(lrows, frows, aprev, A, beta, !skip0, xi, gs);
#pragma unroll
    for (int e = 0; e < D * D; e++) xi_l[e] += (double)xi[e];
#pragma unroll
    for (int d = 0; d < D; d++) g_l[d] += (double)gs[d];
}

// Viterbi forward sweep over one slice (Alg. 4 lines 3-6): backpointers into registers (D <= 4:
// one 16-bit nibble word per step, two steps per u32; D > 4: one u32 per step), returns the slice
// map f(x_end) = state before the slice, accumulates sum (o_t + m_t).
template <int D> __host__ __device__ constexpr int st_bpw(int S) { return D <= 4 ? S / 2 : S; }
template <int D, int S, class RS>
__device__ __forceinline__ uint64_t vit_fwd_slice(const RS rows, int nr, bool t0, const float* LA,
                                                  const float* LP, float* V, double& lp, int& zero_i,
                                                  uint32_t* bpw) {
    uint32_t olo = 0x03020100u, ohi = 0x07060504u;
    zero_i = -1;
    float facc = 0.0f;  // sum of (o_t + m_t) over the slice (<= 64 terms), added to the fp64 total once
#pragma unroll
    for (int i = 0; i < st_bpw<D>(S); i++) bpw[i] = 0u;
#pragma unroll
    for (int i = 0; i < S; i++) {
        if (i < nr) {
            float v[D];
            ld_row<D>(rows(i), v);
            float m = vmax<D>(v);
            if (!(m > neg_inf())) m = 0.0f;
            float Vh[D];
            uint32_t sel = 0;
            const bool first = t0 && i == 0;
            // scores V(k) + LA(k, j): FADD2 over column pairs (even D; same operands, bit-identical)
            float scs[D][D];  // [j][k]
            if (D % 2 == 0 && D <= 4 && !first) {
#pragma unroll
                for (int k = 0; k < D; k++) {
                    const float2 vk = make_float2(V[k], V[k]);
#pragma unroll
                    for (int jj = 0; jj < D / 2; jj++) {
                        const float2 s2 = __fadd2_rn(vk, make_float2(LA[k * D + 2 * jj], LA[k * D + 2 * jj + 1]));
                        scs[2 * jj][k] = s2.x;
                        scs[2 * jj + 1][k] = s2.y;
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < D; j++)
#pragma unroll
                    for (int k = 0; k < D; k++) scs[j][k] = V[k] + (first ? LP[j] : LA[k * D + j]);
            }
#pragma unroll
            for (int j = 0; j < D; j++) {
                float sc[D];
#pragma unroll
                for (int k = 0; k < D; k++) sc[k] = scs[j][k];
                // the max by a 2-input tree keeps the V recursion's critical path short; the argmax
                // (smallest index attaining it: DESIGN.md reading 5) hangs off it
                float best;
                if constexpr (D == 4) best = fmaxf(fmaxf(sc[0], sc[1]), fmaxf(sc[2], sc[3]));
                else best = vmax<D>(sc);
                int arg = D - 1;
#pragma unroll
                for (int k = D - 2; k >= 0; k--) arg = (sc[k] == best) ? k : arg;
                Vh[j] = best + (v[j] - m);
                sel |= (uint32_t)arg << (4 * j);
            }
            float o = vmax<D>(Vh);
            if (!(o > neg_inf())) {
                if (zero_i < 0) zero_i = i;
                o = 0.0f;
            }
#pragma unroll
            for (int j = 0; j < D; j++) V[j] = Vh[j] - o;
            facc += o + m;
            if constexpr (D <= 4) {
                bpw[i >> 1] |= sel << (16 * (i & 1));
                olo = __byte_perm(olo, 0u, sel);
            } else {
                bpw[i] = sel;
                const uint32_t nlo = __byte_perm(olo, ohi, sel & 0xffffu);
                ohi = __byte_perm(olo, ohi, sel >> 16);
                olo = nlo;
            }
        }
    }
    const double dacc = (double)facc;
    lp += dacc;
    uint64_t f = ((uint64_t)ohi << 32) | olo;
    if constexpr (D < 8) f &= (1ull << (8 * D)) - 1ull;
    return f;
}
// Backtrack over one slice from its end state x; returns the state before the slice.
template <int D, int S>
__device__ __forceinline__ int vit_back_slice(const uint32_t* bpw, int nr, int x, int32_t* out) {
#pragma unroll
    for (int i = S - 1; i >= 0; i--) {
        if (i < nr) {
            out[i] = x;
            const uint32_t sel = (D <= 4) ? (bpw[i >> 1] >> (16 * (i & 1))) & 0xffffu : bpw[i];
            x = (int)((sel >> (4 * x)) & 0xfu);
        }
    }
    return x;
}

// ---------------------------------------------------------------------------- the kernel
// grid = G CTAs (one per SM, cooperative), block = NT lanes.  OP 0: smoother, OP 1: Viterbi.
template <int D, int OP>
__global__ void __launch_bounds__(stream_nt(D)) hmm_stream_kernel(const SParams p) {
    constexpr int NT = stream_nt(D);
    constexpr int NW = NT / 32;
    constexpr int S = stream_s(D);
    constexpr int PITCH = stream_pitch(D);
    constexpr int QB = stream_qb(D);
    constexpr int BPW = st_bpw<D>(S);     // backpointer words per slice
    constexpr int BPB = small_bpb(D);     // backpointer bytes per step
    constexpr int NCB = S * BPB / 8;      // 8-B chunks of one lane's backpointer slice
    constexpr bool MP = (OP == 1 || OP == 4);
    constexpr bool STATS = (OP == 2);  // smoother + Baum-Welch E-step statistics
    constexpr bool SYM = (OP >= 3);    // symbol inputs y[T], log_B[D][V]
    constexpr int NN = 2 * NT;
    extern __shared__ __align__(128) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int c = blockIdx.x, G = gridDim.x;
    const int64_t T = p.T, n = p.n, tb = p.t_base;
    const int K = p.K;
    const int mode = p.mode;
    const int64_t a0 = ((int64_t)c * NT + tid) * n;           // lane range [a0, a1)
    const int64_t a1 = (a0 + n < T) ? a0 + n : T;
    const int nsl = (a0 < a1) ? (int)((a1 - a0 + S - 1) / S) : 0;  // real slices of this lane
    auto slice_rows = [&](int k) -> int {
        if (k >= nsl) return 0;
        const int64_t r0 = a0 + (int64_t)k * S;
        return (int)((a1 - r0 < S) ? a1 - r0 : S);
    };

    uint32_t* sync = reinterpret_cast<uint32_t*>(p.ws + p.ws_sync);
    unsigned long long* arrive1 = reinterpret_cast<unsigned long long*>(sync + 0);
    unsigned long long* arrive2 = reinterpret_cast<unsigned long long*>(sync + 2);
    unsigned long long* zero_code = reinterpret_cast<unsigned long long*>(sync + 4);
    uint32_t* done_ctr = sync + 7;
    uint32_t* bad_flag = sync + 8;
    uint8_t* slots = p.ws + p.ws_slots;
    const size_t map_off = align16((size_t)D * D * 4);
    const int sw = (int)(p.slot_bytes / 4);
    uint8_t* myslot = slots + (size_t)c * p.slot_bytes;

    uint8_t* ring = smem + p.L.ring;
    float* tree = reinterpret_cast<float*>(smem + p.L.tree);
    uint64_t* maps = reinterpret_cast<uint64_t*>(smem + p.L.maps);
    int32_t* ends = reinterpret_cast<int32_t*>(smem + p.L.ends);
    float* stage = reinterpret_cast<float*>(smem + p.L.stage);
    uint8_t* qbuf = smem + p.L.qbuf;
    uint64_t* qbar = reinterpret_cast<uint64_t*>(smem + p.L.misc);  // [NW] Q-block barriers
    double* red = reinterpret_cast<double*>(qbar + NW);
    float* cta_pre = reinterpret_cast<float*>(red + NW);
    float* cta_suf = cta_pre + D;
    int* flag = reinterpret_cast<int*>(cta_suf + D);

    unsigned long long* tmr = p.timers ? p.timers + (size_t)c * 16 : nullptr;
#define HMM_STAMP(i) do { if (tmr && tid == 0) tmr[i] = global_ns(); } while (0)
    HMM_STAMP(0);
    if (tmr && tid == 0) {  // slot 13: the SM this CTA runs on (phase profiles per SM)
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        tmr[13] = smid;
    }
    if (tid == 0) {
        for (int w = 0; w < NW; w++) mbar_init(&qbar[w], 1);
        fence_mbar_init();
        flag[0] = -1;
    }
    __syncthreads();

    float A[D * D], pv[D];
#pragma unroll
    for (int e = 0; e < D * D; e++) {
        const float la = __ldg(p.log_A + e);
        A[e] = MP ? la : ex2(la * kLog2e);
    }
#pragma unroll
    for (int d = 0; d < D; d++) {
        const float lp = __ldg(p.log_pi + d);
        pv[d] = MP ? lp : ex2(lp * kLog2e);
    }

    bool bad = false;
    double acc = 0.0;
    int64_t zero_t = INT64_MAX;
    const float* ll = p.log_lik;
    float* tab = reinterpret_cast<float*>(smem + p.L.tab);  // [V][D] = log_B transposed (symbol inputs)
    if constexpr (SYM) {
        for (int e = tid; e < p.V * D; e += NT) {
            const int v = e / D, d = e - v * D;
            const float x = __ldg(p.log_B + d * p.V + v);
            tab[e] = x;
            if (x != x || (x == INFINITY)) bad = true;  // NaN / +inf in log_B (reported like log_lik)
        }
        __syncthreads();
    }
    // lane's slot in ring stage st
    auto slot = [&](int st) -> float* {
        return reinterpret_cast<float*>(ring + (size_t)st * NT * PITCH + (size_t)tid * PITCH);
    };
    // Warp-cooperative slice movement.  A lane's slice is S*D*4 contiguous bytes, but the 32 lanes of
    // a warp are n steps apart, so per-lane bulk copies (UBLKCP takes uniform operands: the compiler
    // serialises them over the lanes) cost ~10 instructions per lane.  Instead the warp moves its 32
    // slices with 16-B per-thread accesses, CPL consecutive threads per lane slice: cp.async (LDGSTS)
    // for loads into the ring, LDS + STG.128 for stores -- fully coalesced segments.  (Plain stores:
    // the evict-first st.global.cs form measured ~10 us slower at T = 1e8.)
    constexpr int CPL = S * D / 4;  // 16-B chunks per full lane slice
    // symbol inputs: the S symbol bytes of a lane slice sit at the END of its row area, so the in-order
    // sweep that overwrites rows with l_t (smoother pass 2) only ever overwrites symbols it has consumed:
    // row i ends at byte 4D(i+1) <= YOFF + i + 1 for every i < S.
    constexpr int YOFF = S * D * 4 - S;
    const int64_t wbase = ((int64_t)c * NT + warp * 32) * n;  // first step of this warp's lane 0
    auto lane_rows = [&](int j, int k) -> int {
        const int64_t rem = T - (wbase + (int64_t)j * n + (int64_t)k * S);
        return rem <= 0 ? 0 : (rem < S ? (int)rem : S);
    };
    // Warp geometry against the sequence end, computed once (warp-uniform): lanes [0, jT) are complete,
    // lane jT (if < 32) holds the end with nfT full slices and a partial slice of remT rows, later lanes
    // are empty.  Slice k then has full lane slices [0, jfull(k)); the warp holding the end of the
    // sequence moves them with the same 16-B copies as a full warp, and only the one partial lane slice
    // (k == nfT) takes the element-wise path.  (A per-slice ballot here cost the last warp ~5 % over
    // the other warps in both passes: the step's tail straggler.)
    const int64_t wrem = T - wbase;
    const int jT = wrem >= 32 * n ? 32 : (wrem <= 0 ? 0 : (int)(wrem / n));
    const int64_t inT = (jT < 32 && wrem > 0) ? wrem - (int64_t)jT * n : 0;
    const int nfT = (int)(inT / S), remT = (int)(inT - (int64_t)nfT * S);
    auto jfull = [&](int k) -> int { return jT == 32 ? 32 : jT + (k < nfT ? 1 : 0); };
    auto warp_full = [&](int k) -> bool { return jfull(k) == 32; };
    // async load of slice k of the warp's lanes into ring stage st (one cp.async group per call)
    auto coop_load = [&](int k, int st) {
        uint8_t* sbase = ring + (size_t)st * NT * PITCH + (size_t)warp * 32 * PITCH;
        if constexpr (SYM) {  // the warp's 32 lane slices of symbols: S bytes each, 4-B chunks, zero-filled
            constexpr int NCY = S / 4;
#pragma unroll
            for (int it = 0; it < NCY; it++) {
                const int q = lane + 32 * it, j = q / NCY, cy = q - j * NCY;
                const int64_t r0 = wbase + (int64_t)j * n + (int64_t)k * S + 4 * cy;
                const int64_t rem = T - r0;
                const uint32_t nb = rem <= 0 ? 0u : (rem >= 4 ? 4u : (uint32_t)rem);
                cp_async4_zfill(sbase + (size_t)j * PITCH + YOFF + 4 * cy, nb ? (const void*)(p.y + r0) : (const void*)p.y,
                                nb);
            }
            cp_async_commit();
            return;
        }
        bool done = false;
        if constexpr ((32 % CPL) == 0) {
            constexpr int LPI = 32 / CPL;
            const int ch = lane % CPL, j0 = lane / CPL;
            const float* src = ll + (wbase + (int64_t)j0 * n + (int64_t)k * S) * D + ch * 4;
            uint8_t* dst = sbase + (size_t)j0 * PITCH + ch * 16;
            if (warp_full(k)) {
#pragma unroll
                for (int it = 0; it < CPL; it++) {
                    cp_async16(dst, src);
                    src += (int64_t)LPI * n * D;
                    dst += LPI * PITCH;
                }
            } else {  // the warp holding the end of the sequence (lanes past the end load nothing)
                const int jp = jfull(k);  // lanes [0, jp) full; lane jp's slice k is partial iff k == nfT
                const int nv = (jp - j0 + LPI - 1) / LPI;  // this thread's chunks in full lane slices
#pragma unroll
                for (int it = 0; it < CPL; it++) {
                    if (it < nv) cp_async16(dst, src);
                    src += (int64_t)LPI * n * D;
                    dst += LPI * PITCH;
                }
                if (k == nfT && remT > 0 && ((jp - j0) % LPI) == 0 && jp >= j0) {
                    const int rem = remT * D - ch * 4;
                    if (rem > 0) {
                        const int f = rem > 4 ? 4 : rem;
                        cp_async16_zfill(sbase + (size_t)jp * PITCH + ch * 16,
                                         ll + (wbase + (int64_t)jp * n + (int64_t)k * S) * D + ch * 4, 4u * f);
                    }
                }
            }
            done = true;
        }
        if (!done) {
            for (int q = lane; q < 32 * CPL; q += 32) {
                const int j = q / CPL, ch = q - j * CPL;
                const int fl = lane_rows(j, k) * D, f0 = ch * 4;
                if (f0 >= fl) continue;
                const float* src = ll + (wbase + (int64_t)j * n + (int64_t)k * S) * D + f0;
                float* dst = reinterpret_cast<float*>(sbase + (size_t)j * PITCH) + f0;
                if (f0 + 4 <= fl) {
                    cp_async16(dst, src);
                } else {
                    for (int f = 0; f < fl - f0; f++) cp_async4(dst + f, src + f);
                }
            }
        }
        cp_async_commit();
    };
    // store slice k of the warp's lanes from SMEM slots (stage base `sb`) to the sequence buffer g
    auto coop_store = [&](int k, const uint8_t* sb, float* g) {
        const uint8_t* sbase = sb + (size_t)warp * 32 * PITCH;
        bool done = false;
        if constexpr ((32 % CPL) == 0) {
            constexpr int LPI = 32 / CPL;
            const int ch = lane % CPL, j0 = lane / CPL;
            float* dst = g + (wbase + (int64_t)j0 * n + (int64_t)k * S) * D + ch * 4;
            const uint8_t* src = sbase + (size_t)j0 * PITCH + ch * 16;
            if (warp_full(k)) {
#pragma unroll
                for (int it = 0; it < CPL; it++) {
                    *reinterpret_cast<float4*>(dst) = *reinterpret_cast<const float4*>(src);
                    dst += (int64_t)LPI * n * D;
                    src += LPI * PITCH;
                }
            } else {  // the warp holding the end of the sequence: full lane slices as above
                const int jp = jfull(k);
                const int nv = (jp - j0 + LPI - 1) / LPI;
#pragma unroll
                for (int it = 0; it < CPL; it++) {
                    if (it < nv) *reinterpret_cast<float4*>(dst) = *reinterpret_cast<const float4*>(src);
                    dst += (int64_t)LPI * n * D;
                    src += LPI * PITCH;
                }
                if (k == nfT && remT > 0 && ((jp - j0) % LPI) == 0 && jp >= j0) {
                    const int rem = remT * D - ch * 4;
                    if (rem > 0) {
                        float* d2 = g + (wbase + (int64_t)jp * n + (int64_t)k * S) * D + ch * 4;
                        const float* s2 = reinterpret_cast<const float*>(sbase + (size_t)jp * PITCH + ch * 16);
                        if (rem >= 4) *reinterpret_cast<float4*>(d2) = *reinterpret_cast<const float4*>(s2);
                        else for (int f = 0; f < rem; f++) d2[f] = s2[f];
                    }
                }
            }
            done = true;
        }
        if (!done) {
            for (int q = lane; q < 32 * CPL; q += 32) {
                const int j = q / CPL, ch = q - j * CPL;
                const int fl = lane_rows(j, k) * D, f0 = ch * 4;
                if (f0 >= fl) continue;
                float* dst = g + (wbase + (int64_t)j * n + (int64_t)k * S) * D + f0;
                const float* src = reinterpret_cast<const float*>(sbase + (size_t)j * PITCH) + f0;
                if (f0 + 4 <= fl) {
                    *reinterpret_cast<float4*>(dst) = *reinterpret_cast<const float4*>(src);
                } else {
                    for (int f = 0; f < fl - f0; f++) dst[f] = src[f];
                }
            }
        }
    };
    auto stage_base = [&](int st) -> uint8_t* { return ring + (size_t)st * NT * PITCH; };
    // row source of slice k in ring stage st; symbol inputs are range-checked once per slice
    auto rsrc = [&](int st, int nr) -> RowSrc<D, SYM> {
        const float* rows = slot(st);
        const uint8_t* ys = reinterpret_cast<const uint8_t*>(rows) + YOFF;
        if constexpr (SYM) {
            if (p.V < 256) {
                const uint32_t vrep = 0x01010101u * (uint32_t)p.V;
                uint32_t badw = 0;
#pragma unroll
                for (int w = 0; w < S / 4; w++)
                    if (4 * w < nr) badw |= __vcmpgeu4(reinterpret_cast<const uint32_t*>(ys)[w], vrep);
                if (badw) bad = true;  // (the zero-filled bytes past the sequence end are symbol 0: valid)
            }
        }
        return RowSrc<D, SYM>{rows, ys, tab};
    };

    const bool do_pass1 = (mode == HMM_MODE_FULL || mode == HMM_MODE_REDUCE);
    float P[D * D];
    // ===================== pass 1: right-to-left fold of the lane (3-stage ring, 2 slices in flight)
    if (do_pass1) {
        mat_identity<D, MP>(P);
        float dexp = 0.0f, chk = 0.0f;  // pending exponent offset of P (sum-product)
        const bool lane_t0 = (tb + a0 == 0) && nsl > 0;
        float* qdst = reinterpret_cast<float*>(p.ws + p.ws_q);
        coop_load(K - 1, 0);
        if (K > 1) coop_load(K - 2, 1); else cp_async_commit();
        for (int it = 0; it < K; it++) {
            const int k = K - 1 - it;
            const int st = it % 3;
            if (it + 2 < K) coop_load(k - 2, (it + 2) % 3); else cp_async_commit();
            const int nr = slice_rows(k);
            if constexpr (!MP) {
                if (nr > 0) {  // Q_k = product of the slices right of k (normalised), warp-contiguous
                    const int qi = k;
                    const float s = pow2_inv(vmax_tree<D * D>(P));
#pragma unroll
                    for (int e = 0; e < D * D; e++) P[e] *= s;
                    dexp = 0.0f;
                    float* q = qdst + (((size_t)c * K + qi) * NT + tid) * (QB / 4);
                    if constexpr ((D * D) % 4 == 0) {
#pragma unroll
                        for (int e = 0; e < D * D; e += 4)
                            *reinterpret_cast<float4*>(q + e) = make_float4(P[e], P[e + 1], P[e + 2], P[e + 3]);
                    } else {
#pragma unroll
                        for (int e = 0; e < D * D; e++) q[e] = P[e];
                    }
                }
            }
            cp_async_wait<2>();
            __syncwarp();
            if (nr > 0) {
                const RowSrc<D, SYM> rows = rsrc(st, nr);
                if constexpr (MP) {
                    mp_fold_back<D, S>(rows, nr, lane_t0 && k == 0, A, pv, P, chk);
                    const float m = vmax<D * D>(P);  // renormalise once per slice (max 0)
                    if (m > neg_inf()) {
#pragma unroll
                        for (int e = 0; e < D * D; e++) P[e] -= m;
                    }
                } else {
                    sp_fold_back<D, S>(rows, nr, lane_t0 && k == 0, A, pv, P, dexp);
                }
            }
            __syncwarp();
        }
        if constexpr (MP) {
            bad |= (chk != chk);
        } else {
            const float s = pow2_inv(vmax_tree<D * D>(P));
#pragma unroll
            for (int e = 0; e < D * D; e++) P[e] *= s;
            const float ck = vsum<D * D>(P);
            bad |= (ck != ck);
        }
        if (mode == HMM_MODE_REDUCE) {  // lane aggregate persisted for the finish / forward call
            float* dst = reinterpret_cast<float*>(p.ws + p.ws_lagg) + ((size_t)c * NT + tid) * (QB / 4);
#pragma unroll
            for (int e = 0; e < D * D; e++) dst[e] = P[e];
        }
    } else if (mode == HMM_MODE_SFINISH || mode == HMM_MODE_VFORWARD) {
        const float* src = reinterpret_cast<const float*>(p.ws + p.ws_lagg) + ((size_t)c * NT + tid) * (QB / 4);
#pragma unroll
        for (int e = 0; e < D * D; e++) P[e] = __ldcg(src + e);
    }
    HMM_STAMP(1);
    if (tmr && lane == 0 && warp == NW - 1) tmr[11] = global_ns();  // last warp done with pass 1
    // the ring is reused by the trees from here: all lanes done reading it
    __syncthreads();

    // ===================== CTA tree over the lane aggregates, grid exchange of the CTA roots
    if (mode != HMM_MODE_VFINISH) {
        tree_store<D>(tree, NN, NT + tid, P);
        __syncthreads();
        tree_up<D, MP>(tree, NT);
        if (do_pass1 && tid < D * D) reinterpret_cast<float*>(myslot)[tid] = tree[tid * NN + 1];
        HMM_STAMP(2);
        if (G > 1 || !do_pass1 || mode == HMM_MODE_REDUCE) {
            if (do_pass1) group_arrive_wait(arrive1, (uint32_t)G);
            HMM_STAMP(3);
            copy_root_slots(stage, slots, G, p.slot_bytes, tid, NT);
            __syncthreads();
        }
        if (mode == HMM_MODE_REDUCE) {
            if (c == 0 && warp == 0) {
                float M[D * D];
                warp_prod<D, MP>(stage, sw, 0, G, M);
                if (lane < D * D) p.agg_out[lane] = M[lane];
            }
        } else if (warp == 0) {
            float M[D * D];
            if (c > 0) warp_prod<D, MP>(stage, sw, 0, c, M);
            if (lane == 0) {
                float u[D], v[D];
#pragma unroll
                for (int d = 0; d < D; d++) u[d] = v[d] = MP ? 0.0f : 1.0f;
                for (int q = 0; q < p.rank; q++) {  // ranks to the left (split phase)
                    float X[D * D];
#pragma unroll
                    for (int e = 0; e < D * D; e++) X[e] = __ldg(p.agg_all + (size_t)q * p.agg_stride + e);
                    vec_mat<D, MP>(u, X, v);
#pragma unroll
                    for (int d = 0; d < D; d++) u[d] = v[d];
                }
                if (c > 0) vec_mat<D, MP>(u, M, v);
#pragma unroll
                for (int d = 0; d < D; d++) cta_pre[d] = v[d];
            }
        } else if (warp == 1 && !MP) {
            float M[D * D];
            if (c < G - 1) warp_prod<D, MP>(stage, sw, c + 1, G, M);
            if (lane == 0) {
                float u[D], v[D];
#pragma unroll
                for (int d = 0; d < D; d++) u[d] = v[d] = 1.0f;
                for (int q = p.world - 1; q > p.rank; q--) {  // ranks to the right
                    float X[D * D];
#pragma unroll
                    for (int e = 0; e < D * D; e++) X[e] = __ldg(p.agg_all + (size_t)q * p.agg_stride + e);
                    mat_vec<D>(X, u, v);
#pragma unroll
                    for (int d = 0; d < D; d++) u[d] = v[d];
                }
                if (c < G - 1) mat_vec<D>(M, u, v);
#pragma unroll
                for (int d = 0; d < D; d++) cta_suf[d] = v[d];
            }
        }
        __syncthreads();
    }
    HMM_STAMP(4);
    const bool do_sweep = (mode == HMM_MODE_FULL || mode == HMM_MODE_SFINISH || mode == HMM_MODE_VFORWARD);
    float cin[D], cout_[D];  // lane carries: forward (alpha / V) and backward (beta)
    if (do_sweep) {
        tree_down<D, MP, !MP>(tree, NT, cta_pre, cta_suf);
#pragma unroll
        for (int d = 0; d < D; d++) {
            cin[d] = tree[d * NN + NT + tid];
            cout_[d] = MP ? 0.0f : tree[(D + d) * NN + NT + tid];
        }
    }
    HMM_STAMP(5);
    __syncthreads();          // tree (ring) dead from here
    fence_proxy_async_smem();  // generic-proxy SMEM accesses before the bulk copies reuse it

    if constexpr (!MP) {
        // ===================== smoother pass 2: left to right; ring stages 0/1 = rows, stage 2 = filtered
        if (do_sweep) {
            float alpha[D];
            {
                const float sm_ = vsum<D>(cin);
                const float r = (sm_ > 0.0f) ? 1.0f / sm_ : 0.0f;
#pragma unroll
                for (int d = 0; d < D; d++) alpha[d] = cin[d] * r;
            }
            float rprod = 1.0f;
            int rexp = 0;
            double msum = 0.0;
            const bool lane_t0 = (tb + a0 == 0) && nsl > 0;
            const uint8_t* qsrc = p.ws + p.ws_q;
            float* frows = slot(2);
            auto issue_q = [&](int k) {  // the warp's 32 Q_k slots, one bulk copy by lane 0
                if (lane == 0) {
                    const uint32_t bytes = 32u * QB;
                    mbar_arrive_expect_tx(&qbar[warp], bytes);
                    bulk_g2s(qbuf + (size_t)warp * 32 * QB, qsrc + (((size_t)c * K + k) * NT + warp * 32) * QB, bytes,
                             &qbar[warp]);
                }
            };
            uint32_t qphase = 0;
            double xi_l[STATS ? D * D : 1], g_l[STATS ? D : 1];
#pragma unroll
            for (int e = 0; e < (STATS ? D * D : 1); e++) xi_l[e] = 0.0;
#pragma unroll
            for (int e = 0; e < (STATS ? D : 1); e++) g_l[e] = 0.0;
            coop_load(0, 0);
            issue_q(0);
            for (int k = 0; k < K; k++) {
                const int st = k & 1;
                if (k + 1 < K) coop_load(k + 1, st ^ 1); else cp_async_commit();
                cp_async_wait<1>();
                __syncwarp();
                mbar_wait(&qbar[warp], qphase);
                qphase ^= 1u;
                const int nr = slice_rows(k);
                float beta[D];
                if (nr > 0) {
                    float Q[D * D];
                    const float* qs = reinterpret_cast<const float*>(qbuf + ((size_t)warp * 32 + lane) * QB);
#pragma unroll
                    for (int e = 0; e < D * D; e++) Q[e] = qs[e];
                    mat_vec<D>(Q, cout_, beta);
                }
                __syncwarp();  // every lane has read its Q_k
                if (k + 1 < K) issue_q(k + 1);
                if (nr > 0) {
                    float* rows = slot(st);
                    float aprev[D];
#pragma unroll
                    for (int d = 0; d < D; d++) aprev[d] = alpha[d];
                    const int zi = sp_alpha_slice<D, S>(rsrc(st, nr), rows, frows, nr, lane_t0 && k == 0, A, pv, alpha,
                                                        rprod, rexp, msum);
                    const int64_t r0 = a0 + (int64_t)k * S;
                    if (zi >= 0 && tb + r0 + zi < zero_t) zero_t = tb + r0 + zi;
                    if constexpr (STATS)
                        sp_beta_slice_stats<D, S>(rows, frows, nr, A, beta, aprev, lane_t0 && k == 0, xi_l, g_l);
                    else
                        sp_beta_slice<D, S>(rows, frows, nr, A, beta);
                }
                __syncwarp();
                if (p.smoothed) coop_store(k, stage_base(st), p.smoothed);
                if (p.filtered) coop_store(k, stage_base(2), p.filtered);
                __syncwarp();
            }
            if (nsl > 0) acc += log((double)vsum<D>(alpha)) - log((double)rprod) - (double)rexp * (double)kLn2 + msum;
            if constexpr (STATS) {  // fixed-order CTA sums of the lanes' fp64 partials -> workspace
                double* cst = reinterpret_cast<double*>(p.ws + p.ws_stats) + (size_t)c * (D * D + D);
                double* rbuf = reinterpret_cast<double*>(ring);  // ring is free after the loop
                __syncthreads();
#pragma unroll
                for (int e = 0; e < D * D + D; e++) {
                    double v = (e < D * D) ? xi_l[e < D * D ? e : 0] : g_l[e >= D * D ? e - D * D : 0];
#pragma unroll
                    for (int o = 16; o >= 1; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
                    if (lane == 0) rbuf[e * NW + warp] = v;
                }
                __syncthreads();
                for (int e = tid; e < D * D + D; e += NT) {
                    double v = 0.0;
                    for (int w = 0; w < NW; w++) v += rbuf[e * NW + w];
                    cst[e] = v;
                }
            }
            if (tmr && lane == 0 && warp == NW - 1) tmr[12] = global_ns();  // last warp done with pass 2
        }
        HMM_STAMP(6);
    } else {
        // ===================== Viterbi pass 2: left to right, backpointers to the workspace
        uint8_t* bpg = p.ws + p.ws_bp;
        uint64_t F = map_identity(D);
        if (do_sweep) {
            float V[D];
#pragma unroll
            for (int d = 0; d < D; d++) V[d] = cin[d];
            const bool lane_t0 = (tb + a0 == 0) && nsl > 0;
            coop_load(0, 0);
            if (K > 1) coop_load(1, 1); else cp_async_commit();
            for (int k = 0; k < K; k++) {
                const int st = k % 3;
                if (k + 2 < K) coop_load(k + 2, (k + 2) % 3); else cp_async_commit();
                cp_async_wait<2>();
                __syncwarp();
                const int nr = slice_rows(k);
                if (nr > 0) {
                    uint32_t bpw[BPW];
                    int zi;
                    const uint64_t f = vit_fwd_slice<D, S>(rsrc(st, nr), nr, lane_t0 && k == 0, A, pv, V, acc, zi, bpw);
                    const int64_t r0 = a0 + (int64_t)k * S;
                    if (zi >= 0 && tb + r0 + zi < zero_t) zero_t = tb + r0 + zi;
                    F = map_compose<D>(F, f);
                    // the slice's rows are consumed: its slot now stages the backpointer words
                    uint2* sb = reinterpret_cast<uint2*>(slot(st));
#pragma unroll
                    for (int w = 0; w < BPW; w += 2) sb[w / 2] = make_uint2(bpw[w], bpw[w + 1]);
                    if (r0 + nr == T) {  // this slice ends the local sequence: x* = argmax V (smallest)
                        int xs = 0;
                        for (int d = D - 1; d >= 0; d--)
                            if (V[d] == 0.0f) xs = d;
                        flag[0] = xs;
                    }
                }
                __syncwarp();
                // warp-cooperative store of the 32 lanes' backpointer slices (8-B chunks, coalesced)
                {
                    const uint8_t* sbase = stage_base(st) + (size_t)warp * 32 * PITCH;
#pragma unroll
                    for (int it = 0; it < NCB; it++) {
                        const int q = lane + 32 * it, j = q / NCB, ch = q - j * NCB;
                        if (j < jfull(k) || (j == jT && k == nfT && remT > 0))  // (lane_rows(j, k) > 0)
                            *reinterpret_cast<uint2*>(bpg + (size_t)(wbase + (int64_t)j * n + (int64_t)k * S) * BPB + ch * 8) =
                                *reinterpret_cast<const uint2*>(sbase + (size_t)j * PITCH + ch * 8);
                    }
                }
                __syncwarp();
            }
            if (mode == HMM_MODE_VFORWARD)
                reinterpret_cast<uint64_t*>(p.ws + p.ws_lmap)[(size_t)c * NT + tid] = F;
        } else if (mode == HMM_MODE_VFINISH) {
            F = __ldcg(reinterpret_cast<const unsigned long long*>(p.ws + p.ws_lmap) + (size_t)c * NT + tid);
        }
        HMM_STAMP(6);
        __syncthreads();
        // CTA map and the end state of every lane
        uint64_t* smaps = reinterpret_cast<uint64_t*>(stage);
        if (mode == HMM_MODE_FULL || mode == HMM_MODE_VFORWARD || mode == HMM_MODE_VFINISH) {
            maps[NT + tid] = F;
            __syncthreads();
            map_tree_up<D>(maps, NT);
        }
        if (mode == HMM_MODE_FULL || mode == HMM_MODE_VFORWARD) {
            if (tid == 0) {
                *reinterpret_cast<uint64_t*>(myslot + map_off) = maps[1];
                if (c == G - 1) *reinterpret_cast<int32_t*>(myslot + map_off + 16) = flag[0];
            }
            if (G > 1) group_arrive_wait(arrive2, (uint32_t)G);
            else __syncthreads();
        }
        if (mode == HMM_MODE_VFORWARD) {
            for (int i = tid; i < G; i += NT)
                smaps[i] = __ldcg(reinterpret_cast<const unsigned long long*>(slots + (size_t)i * p.slot_bytes + map_off));
            __syncthreads();
            if (c == 0 && warp == 0) {
                const uint64_t Fr = warp_compose<D>(smaps, 0, G);
                if (lane == 0) *reinterpret_cast<uint64_t*>(p.rec_out) = Fr;
            }
            if (c == G - 1 && tid == 0) *reinterpret_cast<int32_t*>(p.rec_out + 8) = flag[0];
        }
        const bool do_path = (mode == HMM_MODE_FULL || mode == HMM_MODE_VFINISH);
        if (do_path) {
            int xs = flag[0];
            if (G > 1 || mode == HMM_MODE_VFINISH) {
                for (int i = c + 1 + tid; i < G; i += NT) {
                    smaps[i] = __ldcg(reinterpret_cast<const unsigned long long*>(slots + (size_t)i * p.slot_bytes + map_off));
                    if (i == G - 1) flag[3] = __ldcg(reinterpret_cast<const int*>(slots + (size_t)i * p.slot_bytes + map_off + 16));
                }
                if (mode == HMM_MODE_VFINISH && tid == 0) {
                    int x = *reinterpret_cast<const int32_t*>(p.rec_all + (size_t)(p.world - 1) * 16 + 8);
                    for (int q = p.world - 1; q > p.rank; q--)
                        x = map_apply(*reinterpret_cast<const unsigned long long*>(p.rec_all + (size_t)q * 16), x < 0 ? 0 : x);
                    flag[0] = x;
                }
                __syncthreads();
                xs = (mode == HMM_MODE_VFINISH) ? flag[0] : ((c < G - 1) ? flag[3] : flag[0]);
            }
            if (warp == 0) {
                uint64_t Fs = map_identity(D);
                if (c < G - 1) Fs = warp_compose<D>(smaps, c + 1, G);
                if (lane == 0) flag[1] = map_apply(Fs, xs < 0 ? 0 : xs);
            }
            __syncthreads();
            map_tree_down(maps, ends, NT, flag[1]);
            int x = ends[NT + tid];
            HMM_STAMP(7);
            // ===================== pass 3: backtrack right to left, U slices at a time ("super-slice":
            // ~256 B of path per lane, so every lane's path leaves as full 128-B lines -- 64-B runs
            // scattered over 37k lanes cost DRAM row locality).  Backpointers stream through a 3-stage
            // cp.async ring of 8-B chunks; the path is staged in SMEM and stored with coalesced 16-B
            // stores.
            __syncthreads();  // the map trees above live in the ring region
            constexpr int BPS = S * BPB;                                   // backpointer bytes per lane slice
            constexpr int U_RUN = (256 / (S * 4)) < 1 ? 1 : 256 / (S * 4);
            constexpr int NS3 = 4;                                         // backpointer ring depth
            constexpr int U_FIT = (3 * PITCH - 16) / (NS3 * BPS + S * 4);
            constexpr int U = U_RUN < U_FIT ? U_RUN : U_FIT;              // slices per super-slice
            constexpr int SBS = U * BPS;                                   // backpointer bytes per lane per stage
            constexpr int PPITCH = U * S * 4 + 16;                         // path slot pitch
            static_assert(U >= 1 && NS3 * SBS + PPITCH <= 3 * PITCH, "pass-3 staging exceeds the ring");
            constexpr int CB = (BPS % 16 == 0) ? 16 : 8;                   // copy chunk (never straddles a slice)
            constexpr int NCU = SBS / CB;                                  // chunks per lane per stage
            constexpr int PCU = U * S / 4;                                 // 16-B path chunks per lane
            const int KU = (K + U - 1) / U;
            uint8_t* bring = ring;                              // [NS3][NT][SBS]
            uint8_t* pbuf = ring + (size_t)NS3 * NT * SBS;      // [NT][PPITCH]
            const int64_t lane_end_w = T - wbase;               // steps from this warp's lane 0 to the end
            auto bp_load = [&](int u, int sb) {
                uint8_t* sbase = bring + ((size_t)sb * NT + warp * 32) * SBS;
#pragma unroll
                for (int it = 0; it < NCU; it++) {
                    // whole chunks: the backpointer buffer holds T + S steps, so a chunk that starts before
                    // the sequence end may read past it (those steps are never used)
                    const int q = lane + 32 * it, j = q / NCU, rem = q - j * NCU;
                    const int64_t so = (int64_t)u * U * S + (CB * rem) / BPB;  // step offset inside the lane
                    const bool ok = u >= 0 && so < n && (int64_t)j * n + so < lane_end_w;
                    const uint8_t* src = ok ? bpg + (size_t)(wbase + (int64_t)j * n + (int64_t)u * U * S) * BPB + CB * rem : bpg;
                    if constexpr (CB == 16) cp_async16_zfill(sbase + (size_t)j * SBS + 16 * rem, src, ok ? 16u : 0u);
                    else cp_async8_zfill(sbase + (size_t)j * SBS + 8 * rem, src, ok ? 8u : 0u);
                }
                cp_async_commit();
            };
#pragma unroll 1
            for (int i = 0; i < NS3 - 1; i++) {
                if (i < KU) bp_load(KU - 1 - i, i); else cp_async_commit();
            }
            for (int it = 0; it < KU; it++) {
                const int u = KU - 1 - it;
                const int sb = it % NS3;
                if (it + NS3 - 1 < KU) bp_load(u - (NS3 - 1), (it + NS3 - 1) % NS3); else cp_async_commit();
                cp_async_wait<NS3 - 1>();
                __syncwarp();
                int32_t* ps = reinterpret_cast<int32_t*>(pbuf + (size_t)tid * PPITCH);
                const uint8_t* bsl = bring + ((size_t)sb * NT + tid) * SBS;
                if constexpr (U * BPW <= 32 && BPW % 4 == 0 && BPS % 16 == 0) {
                    // all U slices' words up front (16-B LDS): the backtrack chain never waits on SMEM
                    uint32_t cw[U][BPW];
#pragma unroll
                    for (int kk = 0; kk < U; kk++)
#pragma unroll
                        for (int i = 0; i < BPW; i += 4) {
                            const uint4 v = *reinterpret_cast<const uint4*>(bsl + kk * BPS + 4 * i);
                            cw[kk][i] = v.x;
                            cw[kk][i + 1] = v.y;
                            cw[kk][i + 2] = v.z;
                            cw[kk][i + 3] = v.w;
                        }
#pragma unroll
                    for (int kk = U - 1; kk >= 0; kk--) {
                        const int k = u * U + kk;
                        const int nr = (k < K) ? slice_rows(k) : 0;
                        if (nr > 0) {
                            int32_t out[S];
                            x = vit_back_slice<D, S>(cw[kk], nr, x, out);
#pragma unroll
                            for (int i = 0; i < S; i += 4)
                                *reinterpret_cast<int4*>(ps + kk * S + i) = make_int4(out[i], out[i + 1], out[i + 2], out[i + 3]);
                        }
                    }
                } else {
#pragma unroll 1
                for (int kk = U - 1; kk >= 0; kk--) {
                    const int k = u * U + kk;
                    const int nr = (k < K) ? slice_rows(k) : 0;
                    if (nr > 0) {
                        uint32_t cur[BPW];
                        const uint2* bs = reinterpret_cast<const uint2*>(bsl + kk * BPS);
#pragma unroll
                        for (int i = 0; i < BPW; i += 2) {
                            const uint2 v = bs[i / 2];
                            cur[i] = v.x;
                            cur[i + 1] = v.y;
                        }
                        int32_t out[S];
                        x = vit_back_slice<D, S>(cur, nr, x, out);
#pragma unroll
                        for (int i = 0; i < S; i += 4)
                            *reinterpret_cast<int4*>(ps + kk * S + i) = make_int4(out[i], out[i + 1], out[i + 2], out[i + 3]);
                    }
                }
                }
                __syncwarp();
                // coalesced path stores of the super-slice: 16-B chunks, the sequence's last chunk by words
#pragma unroll
                for (int i2 = 0; i2 < PCU; i2++) {
                    const int q = lane + 32 * i2, j = q / PCU, ch = q - j * PCU;
                    const int64_t so = (int64_t)u * U * S + 4 * ch;                 // step offset inside lane j
                    int64_t lim = lane_end_w - (int64_t)j * n;                      // steps of lane j before T
                    if (lim > n) lim = n;
                    const int64_t nv = lim - so;
                    const int32_t* src = reinterpret_cast<const int32_t*>(pbuf + (size_t)(warp * 32 + j) * PPITCH) + 4 * ch;
                    int32_t* dst = p.path + wbase + (int64_t)j * n + so;
                    if (nv >= 4) {
                        *reinterpret_cast<int4*>(dst) = *reinterpret_cast<const int4*>(src);
                    } else {
                        for (int w = 0; w < nv; w++) dst[w] = src[w];
                    }
                }
                __syncwarp();
            }
        }
        HMM_STAMP(8);
    }

    // ===================== scalars: log Z / log_prob, info (last CTA)
    HMM_STAMP(9);
    if (bad) atomicOr(bad_flag, 1u);
    if (zero_t != INT64_MAX) atomicMax(zero_code, (1ull << 62) - (unsigned long long)zero_t);
    const double part = block_sum<NT>(acc, red);
    if (tid == 0) {
        *reinterpret_cast<double*>(myslot + map_off + 8) = part;
        __threadfence();
        const uint32_t prev = atomicAdd(done_ctr, 1u);
        flag[2] = (prev == (uint32_t)G - 1) ? 1 : 0;
    }
    __syncthreads();
    if (flag[2]) {
        __threadfence();
        double v = 0.0;
        for (int x = tid; x < G; x += NT) v += __ldcg(reinterpret_cast<const double*>(slots + (size_t)x * p.slot_bytes + map_off + 8));
        const double tot = block_sum<NT>(v, red);
        if (tid == 0) {
            if (p.scalar_out) p.scalar_out[0] = tot;
            if constexpr (STATS) {
                const double* cst = reinterpret_cast<const double*>(p.ws + p.ws_stats);
                for (int e = 0; e < D * D + D; e++) {
                    double v = 0.0;
                    for (int x = 0; x < G; x++) v += __ldcg(cst + (size_t)x * (D * D + D) + e);
                    if (e < D * D) p.xi_out[e] = v;
                    else p.gamma_out[e - D * D] = v;
                }
            }
            const uint32_t badf = atomicExch(bad_flag, 0u);
            const unsigned long long zc = atomicExch(zero_code, 0ull);
            int32_t inf = 0;
            if (badf) inf = -1;
            else if (zc) inf = (int32_t)((1ull << 62) - zc + 1ull);
            if (p.info) p.info[0] = inf;
            atomicExch(arrive1, 0ull);
            atomicExch(arrive2, 0ull);
            atomicExch(done_ctr, 0u);
        }
    }
    HMM_STAMP(10);
#undef HMM_STAMP
}

// ---------------------------------------------------------------------------- host launch
template <int D, int OP>
static cudaError_t launch_st(unsigned G, const SParams& sp, cudaStream_t stream) {
    auto kern = hmm_stream_kernel<D, OP>;
    const size_t smem = sp.L.total;
    if (cudaError_t e = ensure_smem_optin(reinterpret_cast<const void*>(kern), smem); e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(G, 1, 1);
    cfg.blockDim = dim3((unsigned)stream_nt(D), 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = G > 1 ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, sp);
}

template <int OP>
static cudaError_t launch_st_op(int D, unsigned G, const SParams& sp, cudaStream_t s) {
    switch (D) {
        case 1: return launch_st<1, OP>(G, sp, s);
        case 2: return launch_st<2, OP>(G, sp, s);
        case 3: return launch_st<3, OP>(G, sp, s);
        case 4: return launch_st<4, OP>(G, sp, s);
        case 5: return launch_st<5, OP>(G, sp, s);
        case 6: return launch_st<6, OP>(G, sp, s);
        case 7: return launch_st<7, OP>(G, sp, s);
        case 8: return launch_st<8, OP>(G, sp, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_stream(int D, int op, unsigned G, const SParams& sp, cudaStream_t s) {
    if (op == 2) return launch_st_op<2>(D, G, sp, s);
    if (op == 3) return launch_st_op<3>(D, G, sp, s);
    if (op == 4) return launch_st_op<4>(D, G, sp, s);
    return op == 0 ? launch_st_op<0>(D, G, sp, s) : launch_st_op<1>(D, G, sp, s);
}

}  // namespace hmm
