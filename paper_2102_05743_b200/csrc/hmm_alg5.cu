// hmm_alg5.cu — the paper-faithful Viterbi variants, 1 <= D <= 8, sm_100a.
//
// (1) Algorithm 5, the parallel max-product algorithm: a forward max-product scan
//     gives the maximum forward potentials log psi~f_k = a-bar_{0:k} (Proposition 2),
//     a reversed scan the maximum backward potentials log psi~b_k = a-bar_{k:T+1} (Proposition 3,
//     PAPER.md:704-710), and line 10 assembles x*_k = argmax_x psi~f_k(x) psi~b_k(x) (Theorem 4 / Eq. 21,
//     PAPER.md:661-669), smallest index on ties.  Eq. 21 is only guaranteed to give one
//     coherent path when the MAP is unique, so SPEC's diagnostic is
//     computed on the device: the Eq. 6 joint log-weight of the assembled path against the per-step
//     optimum (= the MAP weight, Theorem 4) and the number of tied steps.  The production Viterbi
//     (hmm_viterbi) recovers the path from backpointers instead (reading 6).
//
//     Block scan with leaf elements (the "block-wise elements" of PAPER.md:759-760), in three launches:
//       a5_up      thread = leaf of L steps folded into a D x D max-plus aggregate (Def. 5), CTA tree
//                  of NT leaves -> block aggregate;
//       a5_carry   per sequence, the block carries: forward a-bar_{0:k} through the blocks to the left,
//                  backward a-bar_{k:T+1} through the blocks to the right (max-plus vector chains);
//       a5_down    the CTA tree again, carries pushed down to the leaves (forward = prefix,
//                  backward = suffix, Props. 2-3), then per leaf the forward recursion of Lemma 3
//                  (psi~f, kept in SMEM) and the backward recursion (psi~b) with the per-step argmax.
//     a5_weight / a5_final add up the assembled path's joint weight and the MAP weight in a fixed order.
//
// (2) Definition 4, the path-element operator v: elements a~_{i:j} carry the max
//     weight A_{i:j}(x_i, x_j) AND the interior path X^_{i:j}(x_i, x_j); their reduction a~_{0:T+1}
//     holds the MAP weight and the MAP path itself (Theorem 3, Corollary 1).  Memory
//     is D^2 states per covered step, so T <= 1024.  One CTA per sequence
//     reduces the T+1 elements by a balanced pairwise tree (order preserved), values and paths in the
//     workspace (L2-resident).
//
// Both are validation variants: plain, deterministic, not tuned for throughput.
#include <cfloat>
#include <cstdint>
#include <cstring>

#include "../../include/hmmscan.h"
#include "hmm_device.cuh"
#include "hmm_small_ops.cuh"

namespace hmm {

template <int D> __host__ __device__ constexpr int a5_nt() { return D <= 4 ? 256 : 128; }
template <int D> __host__ __device__ constexpr int a5_len() { return D <= 4 ? 16 : 8; }
template <int D> __host__ __device__ constexpr int a5_pitch() { return a5_len<D>() * D + 4; }  // floats per leaf slot
// SoA tree of 2 NT nodes; tree_down keeps the prefix / suffix vectors in elements [0, 2D) of a node
template <int D> __host__ __device__ constexpr int a5_tree_floats() {
    return (D * D > 2 * D ? D * D : 2 * D) * 2 * a5_nt<D>();
}

struct A5Params {
    int64_t T, B;
    int nblk, nwblk;
    float tie_tol;
    const float* log_pi;
    const float* log_A;
    const float* log_lik;
    int32_t* path;
    double* log_prob;
    double* path_weight;
    int64_t* n_tied;
    int32_t* info;
    float* leafagg;  // [B][nblk*NT][D*D]
    float* blkagg;   // [B][nblk][D*D]
    float* blkpre;   // [B][nblk][D]
    float* blksuf;   // [B][nblk][D]
    double* gain;    // [B][nblk]   per-block share of the MAP weight
    double* wpart;   // [B][nwblk]  per-block share of the assembled path's joint weight
    unsigned long long* ctr;  // [B][4]: 2^62 - first impossible step (max; 0 = none), tied steps, bad flag
};

// Cooperative, coalesced load of the block's rows [blk0, blk0 + nsteps) into per-leaf slots (pitch
// a5_pitch floats: 16-B aligned rows, leaf bases spread over the banks).
template <int D>
__device__ void a5_load_rows(float* tile, const float* ll, int64_t blk0, int nsteps) {
    constexpr int LD = a5_len<D>() * D, PITCH = a5_pitch<D>();
    const int nf = nsteps * D;
    const float* src = ll + blk0 * D;
    for (int f = threadIdx.x; f < nf; f += blockDim.x) {
        const int leaf = f / LD, off = f - leaf * LD;
        tile[leaf * PITCH + off] = __ldg(src + f);
    }
    __syncthreads();
}

template <int D>
__device__ __forceinline__ void a5_model(const A5Params& p, float* LA, float* LP) {
#pragma unroll
    for (int e = 0; e < D * D; e++) LA[e] = __ldg(p.log_A + e);
#pragma unroll
    for (int d = 0; d < D; d++) LP[d] = __ldg(p.log_pi + d);
}

// ---------------------------------------------------------------------------- (1) Algorithm 5
template <int D>
__global__ void __launch_bounds__(a5_nt<D>()) a5_up(const A5Params p) {
    constexpr int NT = a5_nt<D>(), L = a5_len<D>(), PITCH = a5_pitch<D>();
    extern __shared__ __align__(16) float sm[];
    float* tile = sm;
    float* tree = sm + NT * PITCH;
    const int tid = threadIdx.x, k = blockIdx.x;
    const int64_t b = blockIdx.y, T = p.T;
    const int64_t blk0 = (int64_t)k * NT * L;
    const int nsteps = (int)((T - blk0 < (int64_t)NT * L) ? T - blk0 : (int64_t)NT * L);
    a5_load_rows<D>(tile, p.log_lik + b * T * D, blk0, nsteps);
    float LA[D * D], LP[D], P[D * D];
    a5_model<D>(p, LA, LP);
    const int li = tid * L;
    const int n = (li < nsteps) ? ((nsteps - li < L) ? nsteps - li : L) : 0;
    bool bad = false;
    if (n > 0) mp_leaf<D>(tile + tid * PITCH, n, blk0 + li == 0, LA, LP, P, bad);
    else mat_identity<D, true>(P);
    if (bad) atomicOr(p.ctr + b * 4 + 2, 1ull);
    float* la_out = p.leafagg + ((size_t)b * p.nblk * NT + (size_t)k * NT + tid) * (D * D);
#pragma unroll
    for (int e = 0; e < D * D; e++) la_out[e] = P[e];
    tree_store<D>(tree, 2 * NT, NT + tid, P);
    __syncthreads();
    tree_up<D, true>(tree, NT);
    if (tid < D * D) p.blkagg[((size_t)b * p.nblk + k) * (D * D) + tid] = tree[tid * 2 * NT + 1];
}

// Block carries, one warp per sequence: lane 0 the forward chain (a-bar_{0:k}, starting from the
// row-constant boundary: any finite vector, here 0), lane 1 the backward chain (a-bar_{k:T+1}, starting
// from psi~b_T = 1, i.e. 0 in the log domain).  Vector chains from a known boundary.
template <int D>
__global__ void a5_carry(const A5Params p) {
    const int64_t b = blockIdx.x;
    const int lane = threadIdx.x;
    const int nb = p.nblk;
    const float* agg = p.blkagg + (size_t)b * nb * (D * D);
    float u[D], v[D], M[D * D];
#pragma unroll
    for (int d = 0; d < D; d++) u[d] = 0.0f;
    if (lane == 0) {
        float* pre = p.blkpre + (size_t)b * nb * D;
        for (int k = 0; k < nb; k++) {
#pragma unroll
            for (int d = 0; d < D; d++) pre[(size_t)k * D + d] = u[d];
            if (k + 1 < nb) {
#pragma unroll
                for (int e = 0; e < D * D; e++) M[e] = agg[(size_t)k * D * D + e];
                vec_mat<D, true>(u, M, v);
#pragma unroll
                for (int d = 0; d < D; d++) u[d] = v[d];
            }
        }
    } else if (lane == 1) {
        float* suf = p.blksuf + (size_t)b * nb * D;
        for (int k = nb - 1; k >= 0; k--) {
#pragma unroll
            for (int d = 0; d < D; d++) suf[(size_t)k * D + d] = u[d];
            if (k > 0) {
#pragma unroll
                for (int e = 0; e < D * D; e++) M[e] = agg[(size_t)k * D * D + e];
                mat_vec_sr<D, true>(M, u, v);
#pragma unroll
                for (int d = 0; d < D; d++) u[d] = v[d];
            }
        }
    }
}

template <int D>
__global__ void __launch_bounds__(a5_nt<D>()) a5_down(const A5Params p) {
    constexpr int NT = a5_nt<D>(), L = a5_len<D>(), PITCH = a5_pitch<D>();
    extern __shared__ __align__(16) float sm[];
    float* tile = sm;
    float* vbuf = sm + NT * PITCH;           // psi~f rows of every leaf (same slot layout)
    float* tree = vbuf + NT * PITCH;
    double* red = reinterpret_cast<double*>(tree + a5_tree_floats<D>());
    const int tid = threadIdx.x, k = blockIdx.x;
    const int64_t b = blockIdx.y, T = p.T;
    const int64_t blk0 = (int64_t)k * NT * L;
    const int nsteps = (int)((T - blk0 < (int64_t)NT * L) ? T - blk0 : (int64_t)NT * L);
    const int NN = 2 * NT;
    // leaf aggregates -> tree (rebuilt) -> carries down the tree (Props. 2-3)
    {
        const float* src = p.leafagg + ((size_t)b * p.nblk * NT + (size_t)k * NT + tid) * (D * D);
        float P[D * D];
#pragma unroll
        for (int e = 0; e < D * D; e++) P[e] = src[e];
        tree_store<D>(tree, NN, NT + tid, P);
    }
    __syncthreads();
    tree_up<D, true>(tree, NT);
    float pre_root[D], suf_root[D];
#pragma unroll
    for (int d = 0; d < D; d++) {
        pre_root[d] = p.blkpre[((size_t)b * p.nblk + k) * D + d];
        suf_root[d] = p.blksuf[((size_t)b * p.nblk + k) * D + d];
    }
    tree_down<D, true, true>(tree, NT, pre_root, suf_root);
    float V[D], W[D];
#pragma unroll
    for (int d = 0; d < D; d++) {
        V[d] = tree[d * NN + NT + tid];
        W[d] = tree[(D + d) * NN + NT + tid];
    }
    __syncthreads();
    a5_load_rows<D>(tile, p.log_lik + b * T * D, blk0, nsteps);
    float LA[D * D], LP[D];
    a5_model<D>(p, LA, LP);
    const int li = tid * L;
    const int n = (li < nsteps) ? ((nsteps - li < L) ? nsteps - li : L) : 0;
    const int64_t t0 = blk0 + li;
    float* rows = tile + tid * PITCH;
    float* vr = vbuf + tid * PITCH;
    double gain = 0.0;
    int64_t zero_t = INT64_MAX;
    unsigned long long tied = 0;
    // Lemma 3 forward recursion from the leaf's forward carry, normalised per step (max 0): the
    // subtracted maxima o_t plus the row maxima m_t add up to this leaf's share of the MAP weight
    for (int i = 0; i < n; i++) {
        float v[D], Vn[D];
        ld_row<D>(rows + i * D, v);
        float m = vmax<D>(v);
        if (!(m > neg_inf())) m = 0.0f;
        if (t0 + i == 0) {
            const float c = vmax<D>(V);
#pragma unroll
            for (int j = 0; j < D; j++) Vn[j] = c + LP[j] + (v[j] - m);
        } else {
#pragma unroll
            for (int j = 0; j < D; j++) {
                float s[D];
#pragma unroll
                for (int q = 0; q < D; q++) s[q] = V[q] + LA[q * D + j];
                Vn[j] = vmax<D>(s) + (v[j] - m);
            }
        }
        float o = vmax<D>(Vn);
        if (!(o > neg_inf())) {
            if (zero_t == INT64_MAX) zero_t = t0 + i;
            o = 0.0f;
        }
#pragma unroll
        for (int j = 0; j < D; j++) V[j] = Vn[j] - o;
        gain += (double)o + (double)m;
        st_row<D>(vr + i * D, V);
    }
    // Lemma 3 backward recursion from the leaf's backward carry; Eq. 21 at every step
    for (int i = n - 1; i >= 0; i--) {
        float f[D], s[D];
        ld_row<D>(vr + i * D, f);
#pragma unroll
        for (int j = 0; j < D; j++) s[j] = f[j] + W[j];
        const float best = vmax<D>(s);
        int x = D - 1;
#pragma unroll
        for (int j = D - 2; j >= 0; j--) x = (s[j] == best) ? j : x;
        float second = neg_inf();
#pragma unroll
        for (int j = 0; j < D; j++) second = (j != x) ? fmaxf(second, s[j]) : second;
        if (D > 1 && best - second <= p.tie_tol) tied++;
        p.path[b * T + t0 + i] = x;
        if (i > 0) {  // psi~b_{t-1}(x) = max_y psi_{t-1,t}(x, y) psi~b_t(y), psi from step t's row
            float v[D], Wn[D];
            ld_row<D>(rows + i * D, v);
            float m = vmax<D>(v);
            if (!(m > neg_inf())) m = 0.0f;
#pragma unroll
            for (int q = 0; q < D; q++) {
                float sc[D];
#pragma unroll
                for (int j = 0; j < D; j++) sc[j] = LA[q * D + j] + (v[j] - m) + W[j];
                Wn[q] = vmax<D>(sc);
            }
            const float mw = vmax<D>(Wn);
#pragma unroll
            for (int q = 0; q < D; q++) W[q] = (mw > neg_inf()) ? Wn[q] - mw : Wn[q];
        }
    }
    // first impossible step: max of 2^62 - t over the leaves (0 = none, so a zeroed workspace is "none")
    if (zero_t != INT64_MAX) atomicMax(p.ctr + b * 4 + 0, (1ull << 62) - (unsigned long long)zero_t);
    if (tied) atomicAdd(p.ctr + b * 4 + 1, tied);
    const double g = block_sum<NT>(gain, red);
    if (tid == 0) p.gain[(size_t)b * p.nblk + k] = g;
}

// Eq. 6 joint log-weight of the assembled path, one step per thread, fp64, fixed-order block sums.
__global__ void __launch_bounds__(256) a5_weight(const A5Params p, int D) {
    __shared__ double red[8];
    const int64_t b = blockIdx.y, T = p.T;
    const int64_t t = (int64_t)blockIdx.x * 256 + threadIdx.x;
    double w = 0.0;
    if (t < T) {
        const int32_t* x = p.path + b * T;
        const int xt = x[t];
        w = (double)__ldg(p.log_lik + (b * T + t) * D + xt);
        w += (t == 0) ? (double)__ldg(p.log_pi + xt) : (double)__ldg(p.log_A + x[t - 1] * D + xt);
    }
    const double s = block_sum<256>(w, red);
    if (threadIdx.x == 0) p.wpart[(size_t)b * p.nwblk + blockIdx.x] = s;
}

__global__ void a5_final(const A5Params p) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= p.B) return;
    double lp = 0.0, w = 0.0;
    for (int k = 0; k < p.nblk; k++) lp += p.gain[(size_t)b * p.nblk + k];
    for (int k = 0; k < p.nwblk; k++) w += p.wpart[(size_t)b * p.nwblk + k];
    unsigned long long* c = p.ctr + b * 4;
    const unsigned long long z = c[0], tied = c[1], bad = c[2];
    int32_t info = 0;
    if (z != 0) {
        const unsigned long long t1 = (1ull << 62) - z + 1;  // first impossible step + 1
        info = (int32_t)(t1 <= 0x7fffffffull ? t1 : 0x7fffffffull);
    }
    else if (bad || lp != lp || w != w) info = -1;
    else if (w < lp - 1e-6 * fmax(1.0, fabs(lp))) info = HMM_INFO_AMBIGUOUS;  // incoherent Eq. 21 assembly
    p.log_prob[b] = lp;
    if (p.path_weight) p.path_weight[b] = w;
    if (p.n_tied) p.n_tied[b] = (int64_t)tied;
    p.info[b] = info;
    c[0] = 0; c[1] = 0; c[2] = 0;  // the workspace is left zeroed
}

// ---------------------------------------------------------------------------- (2) Definition 4
// Level buffers: element q of a level covers base elements [q 2^l, min((q+1) 2^l, T+1)) = [a, e); its
// value block (D x D floats, normalised to max 0, offset kept in fp64) sits at vals + q D^2, its D^2
// interior paths of e - a - 1 states at paths + a D^2 (disjoint, as e - a - 1 < e - a).
struct PEParams {
    int64_t T, B;
    const float* log_pi;
    const float* log_A;
    const float* log_lik;
    int32_t* path;
    double* log_prob;
    int32_t* info;
    uint8_t* ws;
    size_t seq_bytes, o_vals1, o_off0, o_off1, o_path0, o_path1;
};

template <int D>
__global__ void __launch_bounds__(256) pe_reduce(const PEParams p) {
    __shared__ double red[8];
    __shared__ int bad_s;
    const int64_t b = blockIdx.x, T = p.T;
    const int tid = threadIdx.x;
    const int64_t NE = T + 1;  // base elements a~_{0:1}, a~_{1:2}, ..., a~_{T:T+1}
    uint8_t* base = p.ws + (size_t)b * p.seq_bytes;
    float* vals[2] = {reinterpret_cast<float*>(base), reinterpret_cast<float*>(base + p.o_vals1)};
    double* offs[2] = {reinterpret_cast<double*>(base + p.o_off0), reinterpret_cast<double*>(base + p.o_off1)};
    uint8_t* paths[2] = {base + p.o_path0, base + p.o_path1};
    const float* ll = p.log_lik + b * T * D;
    if (tid == 0) bad_s = 0;
    __syncthreads();
    // level 0 (Eq. 19 base elements, log domain, each row shifted by its maximum m_t)
    double msum = 0.0;
    bool bad = false;
    for (int64_t e = tid; e < NE; e += blockDim.x) {
        float* v = vals[0] + e * D * D;
        if (e == T) {
#pragma unroll
            for (int q = 0; q < D * D; q++) v[q] = 0.0f;  // a~_{T:T+1}: psi = 1
        } else {
            float r[D];
#pragma unroll
            for (int j = 0; j < D; j++) r[j] = __ldg(ll + e * D + j);
            float m = vmax<D>(r);
            if (!(m > neg_inf())) m = 0.0f;
            msum += (double)m;
            float chk = 0.0f;
#pragma unroll
            for (int i = 0; i < D; i++)
#pragma unroll
                for (int j = 0; j < D; j++) {
                    const float w = r[j] - m;
                    if (i == 0) chk += w;
                    v[i * D + j] = (e == 0 ? __ldg(p.log_pi + j) : __ldg(p.log_A + i * D + j)) + w;
                }
            bad |= (chk != chk);
        }
        offs[0][e] = 0.0;
    }
    if (bad) atomicOr(&bad_s, 1);
    const double ms = block_sum<256>(msum, red);
    __syncthreads();
    // levels: pair (2q, 2q+1) -> q; an odd last element moves up unchanged
    int cur = 0;
    int64_t n = NE;
    for (int64_t span = 1; n > 1; span <<= 1) {
        const int64_t nn = (n + 1) / 2;
        const float* vin = vals[cur];
        float* vout = vals[cur ^ 1];
        const uint8_t* pin = paths[cur];
        uint8_t* pout = paths[cur ^ 1];
        // values + argmax: one (q, i, k) per task; the normalisation of element q needs all its D^2
        // entries, so a second sweep subtracts the maximum
        for (int64_t task = tid; task < nn * D * D; task += blockDim.x) {
            const int64_t q = task / (D * D);
            const int ik = (int)(task - q * D * D), i = ik / D, kk = ik - i * D;
            const int64_t Lq = 2 * q, Rq = 2 * q + 1;
            const int64_t a = Lq * span;
            const int64_t mid = Rq * span;                        // first base element of the right operand
            const int64_t e = (Rq + 1) * span < NE ? (Rq + 1) * span : NE;
            uint8_t* dst = pout + a * D * D;
            if (Rq >= n) {  // carried over unchanged
                vout[q * D * D + ik] = vin[Lq * D * D + ik];
                const int64_t len = (mid < NE ? mid : NE) - a - 1;
                for (int64_t s = 0; s < len; s++) dst[(size_t)ik * len + s] = pin[a * D * D + (size_t)ik * len + s];
                continue;
            }
            // a~_{a:e}(i,k) = max_j A_{a:mid}(i,j) + A_{mid:e}(j,k);  x^_mid(i,k) = smallest argmax
            float best = neg_inf();
            int xh = 0;
#pragma unroll
            for (int j = 0; j < D; j++) {
                const float s = vin[Lq * D * D + i * D + j] + vin[Rq * D * D + j * D + kk];
                if (s > best) { best = s; xh = j; }
            }
            vout[q * D * D + ik] = best;
            // X^_{a:e}(i,k) = (X^_{a:mid}(i, x^), x^, X^_{mid:e}(x^, k))
            const int64_t lenL = mid - a - 1, lenR = e - mid - 1, len = e - a - 1;
            const uint8_t* sl = pin + a * D * D + (size_t)(i * D + xh) * lenL;
            const uint8_t* sr = pin + mid * D * D + (size_t)(xh * D + kk) * lenR;
            uint8_t* d = dst + (size_t)ik * len;
            for (int64_t s = 0; s < lenL; s++) d[s] = sl[s];
            d[lenL] = (uint8_t)xh;
            for (int64_t s = 0; s < lenR; s++) d[lenL + 1 + s] = sr[s];
        }
        __syncthreads();
        for (int64_t q = tid; q < nn; q += blockDim.x) {
            float* v = vout + q * D * D;
            const int64_t Lq = 2 * q, Rq = 2 * q + 1;
            double off = offs[cur][Lq];
            if (Rq < n) {
                float m = vmax<D * D>(v);
                if (!(m > neg_inf())) m = 0.0f;
#pragma unroll
                for (int e = 0; e < D * D; e++) v[e] -= m;
                off += offs[cur][Rq] + (double)m;
            }
            offs[cur ^ 1][q] = off;
        }
        __syncthreads();
        cur ^= 1;
        n = nn;
    }
    // Corollary 1: a~_{0:T+1} = (MAP weight, x*_{1:T}) for any dummy pair, here (0, 0)
    const uint8_t* fp = paths[cur];
    for (int64_t t = tid; t < T; t += blockDim.x) p.path[b * T + t] = fp[t];
    if (tid == 0) {
        const float top = vals[cur][0];
        const double lp = (double)top + offs[cur][0] + ms;
        p.log_prob[b] = lp;
        p.info[b] = bad_s ? -1 : ((top > neg_inf()) ? 0 : HMM_INFO_NO_PATH);
    }
}

// ---------------------------------------------------------------------------- host side
namespace {
template <int D>
size_t a5_up_smem() { return (size_t)a5_nt<D>() * a5_pitch<D>() * 4 + (size_t)a5_tree_floats<D>() * 4; }
template <int D>
size_t a5_down_smem() { return (size_t)2 * a5_nt<D>() * a5_pitch<D>() * 4 + (size_t)a5_tree_floats<D>() * 4 + 64; }
int64_t cdiv64(int64_t a, int64_t b) { return (a + b - 1) / b; }
size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }

struct A5Layout {
    int nblk = 0, nwblk = 0;
    size_t o_leaf = 0, o_blk = 0, o_pre = 0, o_suf = 0, o_gain = 0, o_wpart = 0, o_ctr = 0, total = 0;
};
A5Layout a5_layout(int D, int64_t T, int64_t B) {
    A5Layout L;
    const int NT = D <= 4 ? 256 : 128, LL = D <= 4 ? 16 : 8;
    L.nblk = (int)cdiv64(T, (int64_t)NT * LL);
    L.nwblk = (int)cdiv64(T, 256);
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = a256(off + bytes); return o; };
    L.o_ctr = take((size_t)B * 4 * 8);
    L.o_leaf = take((size_t)B * L.nblk * NT * D * D * 4);
    L.o_blk = take((size_t)B * L.nblk * D * D * 4);
    L.o_pre = take((size_t)B * L.nblk * D * 4);
    L.o_suf = take((size_t)B * L.nblk * D * 4);
    L.o_gain = take((size_t)B * L.nblk * 8);
    L.o_wpart = take((size_t)B * L.nwblk * 8);
    L.total = off;
    return L;
}
struct PELayout {
    size_t seq = 0, o_vals1 = 0, o_off0 = 0, o_off1 = 0, o_path0 = 0, o_path1 = 0;
};
PELayout pe_layout(int D, int64_t T) {
    PELayout L;
    const size_t NE = (size_t)T + 1, D2 = (size_t)D * D;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = a256(off + bytes); return o; };
    take(NE * D2 * 4);  // vals0 at 0
    L.o_vals1 = take(NE * D2 * 4);
    L.o_off0 = take(NE * 8);
    L.o_off1 = take(NE * 8);
    L.o_path0 = take(NE * D2);
    L.o_path1 = take(NE * D2);
    L.seq = off;
    return L;
}

template <int D>
cudaError_t a5_launch(const A5Params& p, cudaStream_t s) {
    constexpr int NT = a5_nt<D>();
    const size_t su = a5_up_smem<D>(), sd = a5_down_smem<D>();
    if (cudaError_t e = ensure_smem_optin((const void*)a5_up<D>, su); e != cudaSuccess) return e;
    if (cudaError_t e = ensure_smem_optin((const void*)a5_down<D>, sd); e != cudaSuccess) return e;
    const dim3 g((unsigned)p.nblk, (unsigned)p.B);
    a5_up<D><<<g, NT, su, s>>>(p);
    a5_carry<D><<<(unsigned)p.B, 32, 0, s>>>(p);
    a5_down<D><<<g, NT, sd, s>>>(p);
    a5_weight<<<dim3((unsigned)p.nwblk, (unsigned)p.B), 256, 0, s>>>(p, D);
    a5_final<<<(unsigned)cdiv64(p.B, 128), 128, 0, s>>>(p);
    return cudaGetLastError();
}
template <int D>
cudaError_t pe_launch(const PEParams& p, cudaStream_t s) {
    pe_reduce<D><<<(unsigned)p.B, 256, 0, s>>>(p);
    return cudaGetLastError();
}
using A5Fn = cudaError_t (*)(const A5Params&, cudaStream_t);
using PEFn = cudaError_t (*)(const PEParams&, cudaStream_t);
const A5Fn kA5[9] = {nullptr, a5_launch<1>, a5_launch<2>, a5_launch<3>, a5_launch<4>,
                     a5_launch<5>, a5_launch<6>, a5_launch<7>, a5_launch<8>};
const PEFn kPE[9] = {nullptr, pe_launch<1>, pe_launch<2>, pe_launch<3>, pe_launch<4>,
                     pe_launch<5>, pe_launch<6>, pe_launch<7>, pe_launch<8>};
bool al(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }
}  // namespace

size_t variants_workspace_size(int op, int D, int64_t T, int64_t B) {
    if (D < 1 || D > 8 || T < 1 || B < 1 || B > 65535) return 0;
    if (op == HMM_OP_VITERBI_MAXPRODUCT) return a5_layout(D, T, B).total;
    if (op == HMM_OP_VITERBI_PATHELEM) return T > HMM_PATHELEM_MAX_T ? 0 : pe_layout(D, T).seq * (size_t)B;
    return 0;
}

}  // namespace hmm

extern "C" {

hmm_status_t hmm_viterbi_maxproduct(int D, int64_t T, int64_t B, const float* log_pi, const float* log_A,
                                    const float* log_lik, float tie_tol, int32_t* path, double* log_prob,
                                    double* path_weight, int64_t* n_tied, int32_t* info, void* workspace,
                                    size_t workspace_bytes, void* stream) {
    using namespace hmm;
    if (D < 1 || T < 1 || B < 1 || B > 65535) return HMM_ERR_INVALID_VALUE;
    if (D > 8) return HMM_ERR_UNSUPPORTED;
    if (!log_pi || !log_A || !log_lik || !path || !log_prob || !info) return HMM_ERR_INVALID_VALUE;
    if (!al(log_pi, 4) || !al(log_A, 4) || !al(log_lik, 4) || !al(path, 4) || !al(log_prob, 8) || !al(info, 4) ||
        (path_weight && !al(path_weight, 8)) || (n_tied && !al(n_tied, 8)) || !(tie_tol >= 0.0f))
        return HMM_ERR_INVALID_VALUE;
    const A5Layout L = a5_layout(D, T, B);
    if (!workspace || workspace_bytes < L.total || !al(workspace, 256)) return HMM_ERR_WORKSPACE;
    uint8_t* w = static_cast<uint8_t*>(workspace);
    A5Params p;
    std::memset(&p, 0, sizeof(p));
    p.T = T; p.B = B; p.nblk = L.nblk; p.nwblk = L.nwblk; p.tie_tol = tie_tol;
    p.log_pi = log_pi; p.log_A = log_A; p.log_lik = log_lik;
    p.path = path; p.log_prob = log_prob; p.path_weight = path_weight; p.n_tied = n_tied; p.info = info;
    p.leafagg = reinterpret_cast<float*>(w + L.o_leaf);
    p.blkagg = reinterpret_cast<float*>(w + L.o_blk);
    p.blkpre = reinterpret_cast<float*>(w + L.o_pre);
    p.blksuf = reinterpret_cast<float*>(w + L.o_suf);
    p.gain = reinterpret_cast<double*>(w + L.o_gain);
    p.wpart = reinterpret_cast<double*>(w + L.o_wpart);
    p.ctr = reinterpret_cast<unsigned long long*>(w + L.o_ctr);
    const cudaError_t e = kA5[D](p, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? HMM_SUCCESS : HMM_ERR_CUDA;
}

hmm_status_t hmm_viterbi_path_elements(int D, int64_t T, int64_t B, const float* log_pi, const float* log_A,
                                       const float* log_lik, int32_t* path, double* log_prob, int32_t* info,
                                       void* workspace, size_t workspace_bytes, void* stream) {
    using namespace hmm;
    if (D < 1 || T < 1 || B < 1 || B > 65535 || T > HMM_PATHELEM_MAX_T) return HMM_ERR_INVALID_VALUE;
    if (D > 8) return HMM_ERR_UNSUPPORTED;
    if (!log_pi || !log_A || !log_lik || !path || !log_prob || !info) return HMM_ERR_INVALID_VALUE;
    if (!al(log_pi, 4) || !al(log_A, 4) || !al(log_lik, 4) || !al(path, 4) || !al(log_prob, 8) || !al(info, 4))
        return HMM_ERR_INVALID_VALUE;
    const PELayout L = pe_layout(D, T);
    if (!workspace || workspace_bytes < L.seq * (size_t)B || !al(workspace, 256)) return HMM_ERR_WORKSPACE;
    PEParams p;
    std::memset(&p, 0, sizeof(p));
    p.T = T; p.B = B; p.log_pi = log_pi; p.log_A = log_A; p.log_lik = log_lik;
    p.path = path; p.log_prob = log_prob; p.info = info;
    p.ws = static_cast<uint8_t*>(workspace);
    p.seq_bytes = L.seq; p.o_vals1 = L.o_vals1; p.o_off0 = L.o_off0; p.o_off1 = L.o_off1;
    p.o_path0 = L.o_path0; p.o_path1 = L.o_path1;
    const cudaError_t e = kPE[D](p, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? HMM_SUCCESS : HMM_ERR_CUDA;
}

}  // extern "C"
