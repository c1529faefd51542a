// hmm_small.cu — parallel-scan HMM smoother and Viterbi for small state counts (1 <= D <= 8), sm_100a.
//
// The scan of Algorithm 3 / Algorithm 5 is organised as a three-level
// block scan instead of Algorithm 2's element-level Blelloch tree ("block-wise
// elements"):
//
//   level 0  leaf     one thread folds S consecutive elements a_{t-1:t} = psi_t (Def. 3 / Def. 5,
//                     PAPER.md:261-291, 677-691) into a D x D aggregate held in registers;
//   level 1  chunk    the NT leaf aggregates of a chunk are combined by an up-sweep tree in shared
//                     memory (the operator of Def. 3 = matrix product, of Def. 5 = max-plus product);
//   level 2  CTA/grid the chunk roots of a CTA, then the G CTA roots of a sequence, by trees; the
//                     CTA roots are exchanged through global memory behind a grid barrier.
//
// Carries then flow down the same trees as D-vectors (the forward potential a_{0:k}, Thm. 1, and the
// backward potential a_{k:T+1}, Thm. 2 / Props. 2-3), and every thread re-runs its S steps as a
// sequential vector recursion (Alg. 1 / Alg. 4 restricted to the leaf) to emit filtered and smoothed
// marginals (Eq. 14) or Viterbi backpointers (Alg. 4 line 5).  The MAP path is
// recovered by composing per-leaf backpointer maps (exact integer operator, associative) instead of
// Eq. 21's per-step argmax, which is unsafe under ties (reading 6).
//
// Numerics (DESIGN.md §"Numerics"): elements are built on the fly as A(i,j) * exp(ll_t(j) - m_t),
// m_t = max_j ll_t(j), so the T x D x D tensor never exists; leaf products are renormalised every step
// by an exact power of two; log Z = sum_t (log c_t + m_t) over the sequential forward normalisers
// c_t, accumulated per leaf and summed in fp64 in a fixed order.  Max-plus values are normalised by
// subtracting the maximum; log_prob = sum_t (o_t + m_t) likewise.
#include <cfloat>
#include <cstdint>
#include <cstring>

#include "hmm_device.cuh"
#include "hmm_plan.h"

namespace hmm {

// ---------------------------------------------------------------------------- small helpers
template <int D>
__device__ __forceinline__ void ld_row(const float* p, float* v) {
    if constexpr (D == 4) {
        float4 x = *reinterpret_cast<const float4*>(p);
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    } else if constexpr (D == 8) {
        float4 x = *reinterpret_cast<const float4*>(p);
        float4 y = *reinterpret_cast<const float4*>(p + 4);
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w; v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
    } else if constexpr (D == 2) {
        float2 x = *reinterpret_cast<const float2*>(p);
        v[0] = x.x; v[1] = x.y;
    } else {
#pragma unroll
        for (int d = 0; d < D; d++) v[d] = p[d];
    }
}
template <int D>
__device__ __forceinline__ void st_row(float* p, const float* v) {
    if constexpr (D == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    } else if constexpr (D == 8) {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
    } else if constexpr (D == 2) {
        *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
    } else {
#pragma unroll
        for (int d = 0; d < D; d++) p[d] = v[d];
    }
}


// Byte-packed state maps (D <= 8): byte x holds f(x).
__device__ __forceinline__ uint64_t map_identity(int D) {
    uint64_t r = 0;
    for (int x = 0; x < D; x++) r |= (uint64_t)x << (8 * x);
    return r;
}
__device__ __forceinline__ int map_apply(uint64_t f, int x) { return (int)((f >> (8 * x)) & 0xffu); }
// (f o g)(x) = f(g(x))
template <int D>
__device__ __forceinline__ uint64_t map_compose(uint64_t f, uint64_t g) {
    uint64_t r = 0;
#pragma unroll
    for (int x = 0; x < D; x++) r |= (uint64_t)map_apply(f, map_apply(g, x)) << (8 * x);
    return r;
}

// ---------------------------------------------------------------------------- semiring products
// Sum-product (Def. 3): C = L . R (matrix product), renormalised by an exact power of two.
// Max-product (Def. 5, log domain): C = L (max,+) R, normalised by subtracting the maximum.
template <int D, bool MP>
__device__ __forceinline__ void mat_op(const float* Lm, const float* Rm, float* C) {
#pragma unroll
    for (int r = 0; r < D; r++) {
#pragma unroll
        for (int j = 0; j < D; j++) {
            if constexpr (MP) {
                float s[D];
#pragma unroll
                for (int k = 0; k < D; k++) s[k] = Lm[r * D + k] + Rm[k * D + j];
                C[r * D + j] = vmax<D>(s);
            } else {
                float acc = Lm[r * D] * Rm[j];
#pragma unroll
                for (int k = 1; k < D; k++) acc = fmaf(Lm[r * D + k], Rm[k * D + j], acc);
                C[r * D + j] = acc;
            }
        }
    }
    float m = vmax<D * D>(C);
    if constexpr (MP) {
        if (m > neg_inf()) {
#pragma unroll
            for (int e = 0; e < D * D; e++) C[e] -= m;
        }
    } else {
        float s = pow2_inv(m);
#pragma unroll
        for (int e = 0; e < D * D; e++) C[e] *= s;
    }
}
template <int D, bool MP>
__device__ __forceinline__ void mat_identity(float* M) {
#pragma unroll
    for (int r = 0; r < D; r++)
#pragma unroll
        for (int j = 0; j < D; j++) M[r * D + j] = (r == j) ? (MP ? 0.0f : 1.0f) : (MP ? neg_inf() : 0.0f);
}
// row vector x matrix: y(j) = (+)_k v(k) (x) M(k,j)    [forward carry through an aggregate]
template <int D, bool MP>
__device__ __forceinline__ void vec_mat(const float* v, const float* M, float* y) {
#pragma unroll
    for (int j = 0; j < D; j++) {
        if constexpr (MP) {
            float s[D];
#pragma unroll
            for (int k = 0; k < D; k++) s[k] = v[k] + M[k * D + j];
            y[j] = vmax<D>(s);
        } else {
            float acc = v[0] * M[j];
#pragma unroll
            for (int k = 1; k < D; k++) acc = fmaf(v[k], M[k * D + j], acc);
            y[j] = acc;
        }
    }
    float m = vmax<D>(y);
    if constexpr (MP) {
        if (m > neg_inf()) {
#pragma unroll
            for (int j = 0; j < D; j++) y[j] -= m;
        }
    } else {
        float s = pow2_inv(m);
#pragma unroll
        for (int j = 0; j < D; j++) y[j] *= s;
    }
}
// matrix x column vector: y(i) = sum_j M(i,j) v(j)    [backward carry, sum-product only]
template <int D>
__device__ __forceinline__ void mat_vec(const float* M, const float* v, float* y) {
#pragma unroll
    for (int i = 0; i < D; i++) {
        float acc = M[i * D] * v[0];
#pragma unroll
        for (int j = 1; j < D; j++) acc = fmaf(M[i * D + j], v[j], acc);
        y[i] = acc;
    }
    float s = pow2_inv(vmax<D>(y));
#pragma unroll
    for (int i = 0; i < D; i++) y[i] *= s;
}

// ---------------------------------------------------------------------------- SoA trees in SMEM
// Heap layout: node 1 is the root, children 2n and 2n+1, leaves NP..2NP-1 (NP a power of two).
// Element e of node x lives at tree[e * (2*NP) + x] (conflict-free stores, 2-way loads).
template <int D>
__device__ __forceinline__ void tree_load(const float* tree, int NN, int x, float* M) {
#pragma unroll
    for (int e = 0; e < D * D; e++) M[e] = tree[e * NN + x];
}
template <int D>
__device__ __forceinline__ void tree_store(float* tree, int NN, int x, const float* M) {
#pragma unroll
    for (int e = 0; e < D * D; e++) tree[e * NN + x] = M[e];
}
template <int D, bool MP>
__device__ void tree_up(float* tree, int NP) {
    const int NN = 2 * NP;
    const int lane = threadIdx.x & 31;
    for (int n = NP >> 1; n >= 1; n >>= 1) {
        // Wide levels: one thread per product (fewest instructions).  Narrow levels (n*D <= threads):
        // D threads per product, one output row each, so the level latency is one row not a matrix.
        if ((32 % D) == 0 && n * D <= (int)blockDim.x) {
            // the group max comes from xor-shuffles inside the D-lane group (warp-uniform loop so every
            // shuffle has a full mask)
            const int work = n * D;
            for (int base = threadIdx.x & ~31; base < work; base += blockDim.x) {
                const int w = base + lane;
                const bool act = w < work;
                const int x = n + (act ? w / D : 0);
                const int r = w % D;
                float Lr[D], row[D];
#pragma unroll
                for (int k = 0; k < D; k++) Lr[k] = tree[(r * D + k) * NN + 2 * x];
#pragma unroll
                for (int j = 0; j < D; j++) {
                    if constexpr (MP) {
                        float sc[D];
#pragma unroll
                        for (int k = 0; k < D; k++) sc[k] = Lr[k] + tree[(k * D + j) * NN + 2 * x + 1];
                        row[j] = vmax<D>(sc);
                    } else {
                        float acc = Lr[0] * tree[j * NN + 2 * x + 1];
#pragma unroll
                        for (int k = 1; k < D; k++) acc = fmaf(Lr[k], tree[(k * D + j) * NN + 2 * x + 1], acc);
                        row[j] = acc;
                    }
                }
                float m = vmax<D>(row);
#pragma unroll
                for (int o = 1; o < D; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
                if constexpr (MP) {
                    if (m > neg_inf()) {
#pragma unroll
                        for (int j = 0; j < D; j++) row[j] -= m;
                    }
                } else {
                    const float sc = pow2_inv(m);
#pragma unroll
                    for (int j = 0; j < D; j++) row[j] *= sc;
                }
                if (act) {
#pragma unroll
                    for (int j = 0; j < D; j++) tree[(r * D + j) * NN + x] = row[j];
                }
            }
        } else {
            for (int k = threadIdx.x; k < n; k += blockDim.x) {
                const int x = n + k;
                float Lm[D * D], Rm[D * D], C[D * D];
                tree_load<D>(tree, NN, 2 * x, Lm);
                tree_load<D>(tree, NN, 2 * x + 1, Rm);
                mat_op<D, MP>(Lm, Rm, C);
                tree_store<D>(tree, NN, x, C);
            }
        }
        __syncthreads();
    }
}
// Down-sweep of carries.  pre(x) = (left boundary) (x) all leaves left of x's subtree,
// suf(x) = all leaves right of x's subtree (x) (right boundary).  pre is stored in elements
// [0, D) and suf in [D, 2D) of the node (overwriting matrices no longer needed).
template <int D, bool MP, bool SUF>
__device__ void tree_down(float* tree, int NP, const float* pre_root, const float* suf_root) {
    const int NN = 2 * NP;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int d = 0; d < D; d++) {
            tree[d * NN + 1] = pre_root[d];
            if (SUF) tree[(D + d) * NN + 1] = suf_root[d];
        }
    }
    __syncthreads();
    for (int n = 1; n < NP; n <<= 1) {
        if ((32 % D) == 0 && n * D <= (int)blockDim.x) {
            // D threads per node: thread d produces element d of preR = pre (x) M_left and of
            // sufL = M_right (x) suf; group max by xor-shuffles for the normalisation.
            const int work = n * D;
            for (int base = threadIdx.x & ~31; base < work; base += blockDim.x) {
                const int w = base + lane;
                const bool act = w < work;
                const int x = n + (act ? w / D : 0);
                const int d = w % D;
                float pre[D], suf[D];
#pragma unroll
                for (int k = 0; k < D; k++) {
                    pre[k] = tree[k * NN + x];
                    if (SUF) suf[k] = tree[(D + k) * NN + x];
                }
                float pr, sl = 0.0f;
                if constexpr (MP) {
                    float sc[D];
#pragma unroll
                    for (int k = 0; k < D; k++) sc[k] = pre[k] + tree[(k * D + d) * NN + 2 * x];
                    pr = vmax<D>(sc);
                } else {
                    pr = pre[0] * tree[d * NN + 2 * x];
#pragma unroll
                    for (int k = 1; k < D; k++) pr = fmaf(pre[k], tree[(k * D + d) * NN + 2 * x], pr);
                    if (SUF) {
                        sl = tree[(d * D) * NN + 2 * x + 1] * suf[0];
#pragma unroll
                        for (int j = 1; j < D; j++) sl = fmaf(tree[(d * D + j) * NN + 2 * x + 1], suf[j], sl);
                    }
                }
                float mp = pr, ms = sl;
#pragma unroll
                for (int o = 1; o < D; o <<= 1) {
                    mp = fmaxf(mp, __shfl_xor_sync(0xffffffffu, mp, o));
                    if (SUF) ms = fmaxf(ms, __shfl_xor_sync(0xffffffffu, ms, o));
                }
                if constexpr (MP) {
                    if (mp > neg_inf()) pr -= mp;
                } else {
                    pr *= pow2_inv(mp);
                    if (SUF) sl *= pow2_inv(ms);
                }
                __syncwarp();
                if (act) {
                    tree[d * NN + 2 * x] = pre[d];
                    tree[d * NN + 2 * x + 1] = pr;
                    if (SUF) {
                        tree[(D + d) * NN + 2 * x] = sl;
                        tree[(D + d) * NN + 2 * x + 1] = suf[d];
                    }
                }
            }
        } else {
            for (int k = threadIdx.x; k < n; k += blockDim.x) {
                const int x = n + k;
                float pre[D], suf[D], Lm[D * D], Rm[D * D], preR[D], sufL[D];
#pragma unroll
                for (int d = 0; d < D; d++) {
                    pre[d] = tree[d * NN + x];
                    if (SUF) suf[d] = tree[(D + d) * NN + x];
                }
                tree_load<D>(tree, NN, 2 * x, Lm);
                vec_mat<D, MP>(pre, Lm, preR);
                if (SUF) {
                    tree_load<D>(tree, NN, 2 * x + 1, Rm);
                    mat_vec<D>(Rm, suf, sufL);
                }
#pragma unroll
                for (int d = 0; d < D; d++) {
                    tree[d * NN + 2 * x] = pre[d];
                    tree[d * NN + 2 * x + 1] = preR[d];
                    if (SUF) {
                        tree[(D + d) * NN + 2 * x] = sufL[d];
                        tree[(D + d) * NN + 2 * x + 1] = suf[d];
                    }
                }
            }
        }
        __syncthreads();
    }
}
// Map trees (Viterbi backtrack): map(x) = map(2x) o map(2x+1); end(2x+1) = end(x), end(2x) = map(2x+1)(end(x)).
template <int D>
__device__ void map_tree_up(uint64_t* maps, int NP) {
    for (int n = NP >> 1; n >= 1; n >>= 1) {
        for (int k = threadIdx.x; k < n; k += blockDim.x) {
            const int x = n + k;
            maps[x] = map_compose<D>(maps[2 * x], maps[2 * x + 1]);
        }
        __syncthreads();
    }
}
__device__ inline void map_tree_down(const uint64_t* maps, int32_t* ends, int NP, int root_end) {
    if (threadIdx.x == 0) ends[1] = root_end;
    __syncthreads();
    for (int n = 1; n < NP; n <<= 1) {
        for (int k = threadIdx.x; k < n; k += blockDim.x) {
            const int x = n + k;
            const int e = ends[x];
            ends[2 * x + 1] = e;
            ends[2 * x] = map_apply(maps[2 * x + 1], e);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------- warp reductions over
// the G CTA roots of a sequence, staged in shared memory (one slot of `sw` words per CTA).  Lane l
// folds a contiguous group in order, then a fixed shuffle tree; the ordered product of slots
// [lo, hi) is returned in all lanes.
template <int D, bool MP>
__device__ void warp_prod(const float* stage, int sw, int lo, int hi, float* out) {
    const int lane = threadIdx.x & 31;
    const int n = hi - lo;
    const int q = (n + 31) / 32;
    int a = lo + lane * q, e = a + q;
    if (e > hi) e = hi;
    float M[D * D];
    if (a < e) {
#pragma unroll
        for (int k = 0; k < D * D; k++) M[k] = stage[(size_t)a * sw + k];
        for (int s = a + 1; s < e; s++) {
            float X[D * D], C[D * D];
#pragma unroll
            for (int k = 0; k < D * D; k++) X[k] = stage[(size_t)s * sw + k];
            mat_op<D, MP>(M, X, C);
#pragma unroll
            for (int k = 0; k < D * D; k++) M[k] = C[k];
        }
    } else {
        mat_identity<D, MP>(M);
    }
    for (int st = 1; st < 32; st <<= 1) {
        float O[D * D];
#pragma unroll
        for (int k = 0; k < D * D; k++) O[k] = __shfl_down_sync(0xffffffffu, M[k], st);
        if ((lane & (2 * st - 1)) == 0 && lane + st < 32 && lo + (lane + st) * q < hi) {
            float C[D * D];
            mat_op<D, MP>(M, O, C);
#pragma unroll
            for (int k = 0; k < D * D; k++) M[k] = C[k];
        }
    }
#pragma unroll
    for (int k = 0; k < D * D; k++) out[k] = __shfl_sync(0xffffffffu, M[k], 0);
}
template <int D>
__device__ uint64_t warp_compose(const uint64_t* maps, int lo, int hi) {
    const int lane = threadIdx.x & 31;
    const int n = hi - lo;
    const int q = (n + 31) / 32;
    int a = lo + lane * q, e = a + q;
    if (e > hi) e = hi;
    uint64_t f = map_identity(D);
    for (int s = a; s < e; s++) f = map_compose<D>(f, maps[s]);
    for (int st = 1; st < 32; st <<= 1) {
        uint64_t o = __shfl_down_sync(0xffffffffu, f, st);
        if ((lane & (2 * st - 1)) == 0 && lane + st < 32) f = map_compose<D>(f, o);
    }
    return __shfl_sync(0xffffffffu, f, 0);
}

// Deterministic block reduction of one double per thread (fixed shuffle + warp order).
template <int NT>
__device__ double block_sum(double v, double* scratch) {
#pragma unroll
    for (int st = 16; st >= 1; st >>= 1) v += __shfl_down_sync(0xffffffffu, v, st);
    if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < NT / 32; w++) s += scratch[w];
    __syncthreads();
    return s;  // valid in thread 0
}

// ---------------------------------------------------------------------------- tile movement
// Whole-CTA load of nf floats (used for small side arrays): bulk copy of the 16-B aligned body on
// `bar`, ordinary loads for the rest.  Returns after the data is visible to all threads.
__device__ inline void load_floats(float* dst, const float* src, int64_t nf, uint64_t* bar, uint32_t& phase) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(src);
    const bool aligned = (a & 15u) == 0;
    const int64_t body = aligned ? (nf / 4) * 4 : 0;  // floats
    if (body > 0 && threadIdx.x == 0) {
        mbar_arrive_expect_tx(bar, (uint32_t)(body * 4));
        bulk_g2s(dst, src, (uint32_t)(body * 4), bar);
    }
    for (int64_t i = body + threadIdx.x; i < nf; i += blockDim.x) dst[i] = __ldg(src + i);
    if (body > 0) {
        mbar_wait(bar, phase);
        phase ^= 1u;
    }
    __syncthreads();
}

// Chunk tile load split into one piece per warp (warp w's 32 leaves = steps [32Sw, 32S(w+1))), each
// a bulk copy completing on its own mbarrier, so a warp starts folding its leaves as soon as its own
// piece has landed (load overlapped with the leaf products of earlier warps).
struct TileLoad {
    bool bulk;      // false: cooperative loads were used and the tile is complete
};
template <int D>
__device__ inline TileLoad tile_issue(float* tile, const float* src, int nch, int S, uint64_t* mbars, int nw) {
    TileLoad tl;
    tl.bulk = (reinterpret_cast<uintptr_t>(src) & 15u) == 0;
    if (!tl.bulk) {
        for (int64_t i = threadIdx.x; i < (int64_t)nch * D; i += blockDim.x) tile[i] = __ldg(src + i);
        __syncthreads();
        return tl;
    }
    if (threadIdx.x == 0) {
        for (int w = 0; w < nw; w++) {
            const int s0 = 32 * S * w;
            if (s0 >= nch) break;
            const int s1 = (s0 + 32 * S < nch) ? s0 + 32 * S : nch;
            const uint32_t body = ((uint32_t)(s1 - s0) * D * 4u) & ~15u;
            if (body) {
                mbar_arrive_expect_tx(&mbars[w], body);
                bulk_g2s(tile + (size_t)s0 * D, src + (size_t)s0 * D, body, &mbars[w]);
            }
        }
    }
    return tl;
}
// Warp w waits for its piece (+ loads the ragged tail of the last piece itself).
template <int D>
__device__ inline void tile_wait(const TileLoad& tl, float* tile, const float* src, int nch, int S, uint64_t* mbars,
                                 uint32_t& wphase) {
    if (!tl.bulk) return;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s0 = 32 * S * w;
    if (s0 >= nch) return;
    const int s1 = (s0 + 32 * S < nch) ? s0 + 32 * S : nch;
    const uint32_t nf = (uint32_t)(s1 - s0) * D;
    const uint32_t body = nf & ~3u;
    if (body) {
        mbar_wait(&mbars[w], wphase);
        wphase ^= 1u;
    }
    for (uint32_t i = body + lane; i < nf; i += 32) tile[(size_t)s0 * D + i] = __ldg(src + (size_t)s0 * D + i);
    __syncwarp();
}
// Warp-cooperative store of nw 32-bit words from smem (written by this warp) to global: one bulk
// store (UBLKCP) for the 16-B aligned body issued by lane 0, ordinary stores for the rest.
__device__ inline void warp_store(void* dst_, const void* src_, int64_t nw) {
    uint32_t* dst = reinterpret_cast<uint32_t*>(dst_);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(src_);
    const int lane = threadIdx.x & 31;
    const bool aligned = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15u) == 0;
    const int64_t body = aligned ? (nw / 4) * 4 : 0;
    fence_proxy_async_smem();
    __syncwarp();
    if (body > 0 && lane == 0) {
        bulk_s2g(dst, src, (uint32_t)(body * 4));
        bulk_commit();
    }
    for (int64_t i = body + lane; i < nw; i += 32) dst[i] = src[i];
}
// Before shared memory read by this warp's bulk stores is overwritten (or the CTA exits).
__device__ inline void warp_store_wait() {
    if ((threadIdx.x & 31) == 0) bulk_wait_all();
    __syncwarp();
}

// ---------------------------------------------------------------------------- leaf kernels
// Sum-product leaf: P = psi_{t0} psi_{t0+1} ... (n >= 1 elements), renormalised every step.
// If write_l, overwrites the tile rows with l_t = exp(ll_t - m_t) (reused by the sweeps).
template <int D>
__device__ __forceinline__ void sp_leaf(float* rows, int n, bool t0, const float* A, const float* pi, float* P,
                                        double& msum, bool write_l, bool acc_m, bool& bad) {
    float s = 1.0f;
    for (int i = 0; i < n; i++) {
        float v[D], l[D];
        ld_row<D>(rows + i * D, v);
        const float m = vmax<D>(v);
        if (m > neg_inf()) {
            if (acc_m) msum += (double)m;
#pragma unroll
            for (int j = 0; j < D; j++) l[j] = ex2((v[j] - m) * kLog2e);  // NaN / +inf propagate to P
        } else {
            const float sv = vsum<D>(v);  // all -inf (impossible step) or NaN among -inf
            bad |= (sv != sv);
#pragma unroll
            for (int j = 0; j < D; j++) l[j] = 0.0f;
        }
        if (write_l) st_row<D>(rows + i * D, l);
        float cs[D];
#pragma unroll
        for (int j = 0; j < D; j++) cs[j] = l[j] * s;
        if (i == 0) {
#pragma unroll
            for (int r = 0; r < D; r++)
#pragma unroll
                for (int j = 0; j < D; j++) P[r * D + j] = (t0 ? pi[j] : A[r * D + j]) * cs[j];
        } else {
#pragma unroll
            for (int r = 0; r < D; r++) {
                float q[D];
#pragma unroll
                for (int j = 0; j < D; j++) {
                    float acc = P[r * D] * A[j];
#pragma unroll
                    for (int k = 1; k < D; k++) acc = fmaf(P[r * D + k], A[k * D + j], acc);
                    q[j] = acc * cs[j];
                }
#pragma unroll
                for (int j = 0; j < D; j++) P[r * D + j] = q[j];
            }
        }
        s = pow2_inv(vmax<D * D>(P));
    }
#pragma unroll
    for (int e = 0; e < D * D; e++) P[e] *= s;
    const float chk = vsum<D * D>(P);  // a NaN or +inf input anywhere in the leaf leaves a NaN here
    bad |= (chk != chk);
}

// Max-product leaf (log domain): P = psi~_{t0} (max,+) ... ; values shifted by -m_t per step,
// normalised (max 0) at the end.
template <int D>
__device__ __forceinline__ void mp_leaf(const float* rows, int n, bool t0, const float* LA, const float* LP, float* P,
                                        bool& bad) {
    float chk = 0.0f;
    for (int i = 0; i < n; i++) {
        float v[D], w[D];
        ld_row<D>(rows + i * D, v);
        float m = vmax<D>(v);
        if (!(m > neg_inf())) m = 0.0f;
#pragma unroll
        for (int j = 0; j < D; j++) w[j] = v[j] - m;
        chk += vsum<D>(w);  // NaN iff a NaN / +inf input (max-plus itself drops NaNs)
        if (i == 0) {
#pragma unroll
            for (int r = 0; r < D; r++)
#pragma unroll
                for (int j = 0; j < D; j++) P[r * D + j] = (t0 ? LP[j] : LA[r * D + j]) + w[j];
        } else {
#pragma unroll
            for (int r = 0; r < D; r++) {
                float q[D];
#pragma unroll
                for (int j = 0; j < D; j++) {
                    float s[D];
#pragma unroll
                    for (int k = 0; k < D; k++) s[k] = P[r * D + k] + LA[k * D + j];
                    q[j] = vmax<D>(s) + w[j];
                }
#pragma unroll
                for (int j = 0; j < D; j++) P[r * D + j] = q[j];
            }
        }
    }
    float m = vmax<D * D>(P);
    if (m > neg_inf()) {
#pragma unroll
        for (int e = 0; e < D * D; e++) P[e] -= m;
    }
    bad |= (chk != chk);
}

// ---------------------------------------------------------------------------- sweeps
// Forward filter over one leaf (Alg. 1 forward pass restricted to the leaf, started from the scan
// carry alpha = a_{0:t0-1} normalised to sum 1): writes filtered rows and adds this leaf's share of
// log Z.  With alpha_t = (alpha_{t-1} psi_t) * r_t, the exact telescoping is
//   log sum(alpha_in . P_leaf) = log sum(alpha_end) - sum_t log r_t,
// so the multipliers actually applied (r_t = rcp(c_t), rounding included) are accumulated, never c_t:
// a biased reciprocal cannot drift log Z.  Returns the first zero-mass index in the leaf, or -1.
template <int D>
__device__ __forceinline__ int sp_alpha(float* lrows, float* frows, int n, bool t0, const float* A, const float* pi,
                                        float* alpha, double& logz, bool from_ll) {
    float rprod = 1.0f;
    int rexp = 0;
    int zero_i = -1;
    double msum = 0.0;
    for (int i = 0; i < n; i++) {
        float l[D];
        ld_row<D>(lrows + i * D, l);
        if (from_ll) {
            const float m = vmax<D>(l);
            if (m > neg_inf()) {
                msum += (double)m;
#pragma unroll
                for (int j = 0; j < D; j++) l[j] = ex2((l[j] - m) * kLog2e);
            } else {
#pragma unroll
                for (int j = 0; j < D; j++) l[j] = 0.0f;
            }
            st_row<D>(lrows + i * D, l);
        }
        float ah[D];
        if (t0 && i == 0) {
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
        if (!(c > 0.0f) && zero_i < 0) zero_i = i;
        const float r = rcp(c);
#pragma unroll
        for (int j = 0; j < D; j++) alpha[j] = ah[j] * r;
        st_row<D>(frows + i * D, alpha);
        // running product of the applied multipliers, exponent split off exactly
        rprod *= r;
        const uint32_t bits = __float_as_uint(rprod);
        rexp += (int)((bits >> 23) & 0xffu) - 127;
        rprod = __uint_as_float((bits & 0x807fffffu) | 0x3f800000u);
    }
    logz += log((double)vsum<D>(alpha)) - log((double)rprod) - (double)rexp * (double)kLn2 + msum;
    return zero_i;
}

// Backward pass over one leaf (Alg. 1 backward restricted to the leaf) combined with Eq. 14:
// smoothed_t = alpha_t * beta_t / Z_t, written over the l rows.
template <int D>
__device__ __forceinline__ void sp_beta(float* lrows, const float* frows, int n, const float* A, float* beta) {
    for (int i = n - 1; i >= 0; i--) {
        float l[D], a[D], g[D];
        ld_row<D>(lrows + i * D, l);
        ld_row<D>(frows + i * D, a);
#pragma unroll
        for (int j = 0; j < D; j++) g[j] = a[j] * beta[j];
        const float z = rcp(vsum<D>(g));
#pragma unroll
        for (int j = 0; j < D; j++) g[j] *= z;
        st_row<D>(lrows + i * D, g);
        if (i > 0) {
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
            const float s = pow2_inv(vmax<D>(bn));
#pragma unroll
            for (int r = 0; r < D; r++) beta[r] = bn[r] * s;
        }
    }
}

// Viterbi forward sweep over one leaf (Alg. 4 lines 3-6, started from the max-product carry V).
// Writes one backpointer word per step (nibble j = u_{t-1}(j)), returns the leaf map
// f(x_end) = state before the leaf, accumulates sum (o_t + m_t).
template <int D>
__device__ __forceinline__ uint64_t vit_sweep(const float* rows, void* bprow, int n, bool t0, const float* LA,
                                              const float* LP, float* V, double& lp, int& zero_i) {
    uint32_t olo = 0x03020100u, ohi = 0x07060504u;  // identity map bytes
    zero_i = -1;
    double acc = 0.0;
    for (int i = 0; i < n; i++) {
        float v[D];
        ld_row<D>(rows + i * D, v);
        float m = vmax<D>(v);
        if (!(m > neg_inf())) m = 0.0f;
        float Vh[D];
        uint32_t sel = 0;
#pragma unroll
        for (int j = 0; j < D; j++) {
            const bool first = t0 && i == 0;
            float best = V[0] + (first ? LP[j] : LA[j]);
            int arg = 0;
#pragma unroll
            for (int k = 1; k < D; k++) {
                const float sc = V[k] + (first ? LP[j] : LA[k * D + j]);
                if (sc > best) { best = sc; arg = k; }
            }
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
        acc += (double)(o + m);
        if constexpr (D <= 4) {
            reinterpret_cast<uint16_t*>(bprow)[i] = (uint16_t)sel;
            olo = __byte_perm(olo, 0u, sel);
        } else {
            reinterpret_cast<uint32_t*>(bprow)[i] = sel;
            const uint32_t nlo = __byte_perm(olo, ohi, sel & 0xffffu);
            ohi = __byte_perm(olo, ohi, sel >> 16);
            olo = nlo;
        }
    }
    lp += acc;
    uint64_t f = ((uint64_t)ohi << 32) | olo;
    if constexpr (D < 8) f &= (1ull << (8 * D)) - 1ull;
    return f;
}
template <int D>
__device__ __forceinline__ void vit_backtrack(const void* bprow, int32_t* out, int n, int x) {
    for (int i = n - 1; i >= 0; i--) {
        out[i] = x;
        const uint32_t sel = (D <= 4) ? (uint32_t)reinterpret_cast<const uint16_t*>(bprow)[i]
                                      : reinterpret_cast<const uint32_t*>(bprow)[i];
        x = (int)((sel >> (4 * x)) & 0xfu);
    }
}

// ---------------------------------------------------------------------------- the kernel
// grid = (G, B): CTA c of sequence b.  block = NT threads.  OP 0: smoother, OP 1: Viterbi.
template <int D, int OP>
__global__ void __launch_bounds__(small_nt(D)) hmm_small_kernel(const KParams p) {
    constexpr int NT = small_nt(D);
    constexpr int NW = NT / 32;
    constexpr bool MP = (OP == 1);
    extern __shared__ __align__(128) uint8_t smem[];
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int c = blockIdx.x, G = gridDim.x;
    const int64_t b = blockIdx.y;
    const int64_t T = p.T;
    const int64_t cta0 = (int64_t)c * p.R;
    const int64_t cta1 = (cta0 + p.R < T) ? cta0 + p.R : T;
    const int nchunks = (int)((cta1 - cta0 + p.chunk - 1) / p.chunk);
    const int S = p.S;
    const bool fused = p.fused != 0;
    const int mode = p.mode;
    const bool do_pass1 = (mode == HMM_MODE_FULL || mode == HMM_MODE_REDUCE);
    const int64_t tb = p.t_base;  // global index of local step 0 (split-phase ranks)

    // per-sequence sync block (64 B): [0] u64 arrivals of exchange 1, [2] u64 arrivals of exchange 2,
    // [4] u64 impossible-step code, [6] epoch, [7] done counter, [8] bad-input flag
    uint32_t* sync = reinterpret_cast<uint32_t*>(p.ws + p.ws_sync + (size_t)b * 64);
    unsigned long long* arrive1 = reinterpret_cast<unsigned long long*>(sync + 0);
    unsigned long long* arrive2 = reinterpret_cast<unsigned long long*>(sync + 2);
    unsigned long long* zero_code = reinterpret_cast<unsigned long long*>(sync + 4);
    uint8_t* slots = p.ws + p.ws_slots + (size_t)b * G * p.slot_bytes;
    const size_t map_off = align16((size_t)D * D * 4);
    const int sw = (int)(p.slot_bytes / 4);  // slot stride in words
    uint8_t* myslot = slots + (size_t)c * p.slot_bytes;
    const float* ll_seq = p.log_lik + (size_t)b * T * D;

    float* tile = reinterpret_cast<float*>(smem + p.L.tile);
    float* carr = reinterpret_cast<float*>(smem + p.L.carr);
    float* tree = reinterpret_cast<float*>(smem + p.L.tree);
    float* stage = reinterpret_cast<float*>(smem + p.L.stage);
    uint64_t* mbars = reinterpret_cast<uint64_t*>(smem + p.L.misc);  // NW piece barriers + 1 aux
    uint64_t* mbar_aux = mbars + NW;
    double* red = reinterpret_cast<double*>(smem + p.L.misc + 8 * (NW + 1));
    float* cta_pre = reinterpret_cast<float*>(red + NT / 32);
    float* cta_suf = cta_pre + D;
    int* flag = reinterpret_cast<int*>(cta_suf + D);

    unsigned long long* tmr = p.timers ? p.timers + ((size_t)b * G + c) * 16 : nullptr;
#define HMM_STAMP(i) do { if (tmr && tid == 0) tmr[i] = global_ns(); } while (0)
    HMM_STAMP(0);
    uint32_t* done_ctr = sync + 7;
    uint32_t* bad_flag = sync + 8;
    if (tid == 0) {
        for (int w = 0; w <= NW; w++) mbar_init(&mbars[w], 1);
        fence_mbar_init();
        flag[0] = -1;
    }
    __syncthreads();
    uint32_t wphase = 0, aux_phase = 0;

    // model in registers
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
    double acc = 0.0;            // log Z / log_prob partial of this thread
    int64_t zero_t = INT64_MAX;  // smallest impossible step seen by this thread

    // leaf aggregate of this thread for chunk [ch0, ch0+nch): load (pipelined per warp), fold, store leaf
    auto leaf_pass = [&](int64_t ch0, int nch, bool write_l, bool acc_m, bool& badf) {
        const float* src = ll_seq + ch0 * D;
        fence_proxy_async_smem();  // earlier generic-proxy smem writes before the bulk copies overwrite them
        __syncthreads();
        const TileLoad tl = tile_issue<D>(tile, src, nch, S, mbars, NW);
        tile_wait<D>(tl, tile, src, nch, S, mbars, wphase);
        HMM_STAMP(11);
        const int li = tid * S;
        const int ln = (li < nch) ? ((nch - li < S) ? nch - li : S) : 0;
        float P[D * D];
        if (ln > 0) {
            if constexpr (MP)
                mp_leaf<D>(tile + li * D, ln, tb + ch0 + li == 0, A, pv, P, badf);
            else
                sp_leaf<D>(tile + li * D, ln, tb + ch0 + li == 0, A, pv, P, acc, write_l, acc_m, badf);
        } else {
            mat_identity<D, MP>(P);
        }
        HMM_STAMP(12);
        tree_store<D>(tree, 2 * NT, NT + tid, P);
        __syncthreads();
        HMM_STAMP(13);
        tree_up<D, MP>(tree, NT);
    };

    // ===================== pass 1: leaf aggregates -> chunk roots (split-phase finish calls reuse the
    // chunk roots the reduce call left in the workspace)
    for (int k = 0; do_pass1 && k < nchunks; k++) {
        const int64_t ch0 = cta0 + (int64_t)k * p.chunk;
        const int nch = (int)(((ch0 + p.chunk < cta1) ? ch0 + p.chunk : cta1) - ch0);
        leaf_pass(ch0, nch, fused, true, bad);
        HMM_STAMP(1);
        if (!fused) {
            float* dst = reinterpret_cast<float*>(p.ws + p.ws_chunk + ((size_t)(b * G + c) * p.K + k) * p.chunk_slot);
            if (tid < D * D) dst[tid] = tree[tid * 2 * NT + 1];
            __syncthreads();
        }
    }

    // ===================== CTA root (fused: the chunk tree root; else a tree over chunk roots)
    if (!fused && mode != HMM_MODE_VFINISH) {
        const int NN = 2 * p.KP;
        for (int x = tid; x < p.KP; x += NT) {
            float M[D * D];
            if (x < nchunks) {
                const float* src = reinterpret_cast<const float*>(p.ws + p.ws_chunk +
                                                                  ((size_t)(b * G + c) * p.K + x) * p.chunk_slot);
#pragma unroll
                for (int e = 0; e < D * D; e++) M[e] = src[e];
            } else {
                mat_identity<D, MP>(M);
            }
            tree_store<D>(tree, NN, p.KP + x, M);
        }
        __syncthreads();
        tree_up<D, MP>(tree, p.KP);
    }
    const int NNroot = fused ? 2 * NT : 2 * p.KP;

    // ===================== cross-CTA exchange: publish the root, barrier, stage all roots in SMEM,
    // warp 0 folds the roots to the left (forward carry), warp 1 the roots to the right (backward).
    // Finish calls of the split-phase path find the roots already published by their reduce call.
    if (mode != HMM_MODE_VFINISH) {
        if (do_pass1 && tid < D * D) reinterpret_cast<float*>(myslot)[tid] = tree[tid * NNroot + 1];
        HMM_STAMP(2);
        if (G > 1 || !do_pass1 || mode == HMM_MODE_REDUCE) {
            if (do_pass1) group_arrive_wait(arrive1, (uint32_t)G);  // (G == 1: just a CTA barrier)
            HMM_STAMP(3);
            // copy all G roots into SMEM: one round of independent loads
            for (int i = tid; i < G; i += NT) {
                const float* src = reinterpret_cast<const float*>(slots + (size_t)i * p.slot_bytes);
                float v[D * D];
#pragma unroll
                for (int e = 0; e < D * D; e++) v[e] = __ldcg(src + e);
#pragma unroll
                for (int e = 0; e < D * D; e++) stage[(size_t)i * sw + e] = v[e];
            }
            __syncthreads();
        }
        if (mode == HMM_MODE_REDUCE) {
            // the rank aggregate = ordered product of all G CTA roots
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
                // rank carry (split phase): fold the aggregates of the ranks to the left
                for (int q = 0; q < p.rank; q++) {
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
                for (int q = p.world - 1; q > p.rank; q--) {
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
    // carries per chunk (non-fused) or per leaf (fused)
    if (!do_sweep) {
    } else if (!fused) {
        tree_down<D, MP, !MP>(tree, p.KP, cta_pre, cta_suf);
        const int NN = 2 * p.KP;
        for (int x = tid; x < nchunks; x += NT) {
#pragma unroll
            for (int d = 0; d < D; d++) {
                carr[x * 2 * D + d] = tree[d * NN + p.KP + x];
                if (!MP) carr[x * 2 * D + D + d] = tree[(D + d) * NN + p.KP + x];
            }
        }
        __syncthreads();
    } else {
        tree_down<D, MP, !MP>(tree, NT, cta_pre, cta_suf);
    }

    // this warp's rows of a chunk: [32 S warp, 32 S (warp+1)) clipped to nch
    auto warp_rows = [&](int nch, int& r0, int& nr) {
        r0 = 32 * S * warp;
        int r1 = r0 + 32 * S;
        if (r1 > nch) r1 = nch;
        nr = (r1 > r0) ? r1 - r0 : 0;
    };

    if constexpr (OP == 0) {
        // ===================== smoother pass 2 (chunks in reverse order: the tail is still in L2)
        float* filt = reinterpret_cast<float*>(smem + p.L.regB);
        for (int k = nchunks - 1; do_sweep && k >= 0; k--) {
            const int64_t ch0 = cta0 + (int64_t)k * p.chunk;
            const int nch = (int)(((ch0 + p.chunk < cta1) ? ch0 + p.chunk : cta1) - ch0);
            const int li = tid * S;
            const int ln = (li < nch) ? ((nch - li < S) ? nch - li : S) : 0;
            const bool t0 = (tb + ch0 + li == 0);
            if (!fused) {
                bool dbad = false;
                // (a split-phase finish skipped pass 1, so it accumulates sum m_t here)
                leaf_pass(ch0, nch, true, mode == HMM_MODE_SFINISH, dbad);
                tree_down<D, false, true>(tree, NT, carr + k * 2 * D, carr + k * 2 * D + D);
            }
            float alpha[D], beta[D];
#pragma unroll
            for (int d = 0; d < D; d++) {
                alpha[d] = tree[d * 2 * NT + NT + tid];
                beta[d] = tree[(D + d) * 2 * NT + NT + tid];
            }
            {
                const float s = vsum<D>(alpha);
                const float r = (s > 0.0f) ? 1.0f / s : 0.0f;
#pragma unroll
                for (int d = 0; d < D; d++) alpha[d] *= r;
            }
            __syncthreads();  // the tree (in regB) is dead from here: filtered rows overwrite it
            HMM_STAMP(5);
            if (tmr && tid == 0) tmr[14] = clock64();
            if (ln > 0) {
                const int zi = sp_alpha<D>(tile + li * D, filt + li * D, ln, t0, A, pv, alpha, acc, false);
                if (zi >= 0 && tb + ch0 + li + zi < zero_t) zero_t = tb + ch0 + li + zi;
            }
            int r0, nr;
            warp_rows(nch, r0, nr);
            if (p.filtered && nr > 0)
                warp_store(p.filtered + ((size_t)b * T + ch0 + r0) * D, filt + (size_t)r0 * D, (int64_t)nr * D);
            if (tmr && tid == 0) tmr[15] = clock64();
            HMM_STAMP(6);
            if (ln > 0) sp_beta<D>(tile + li * D, filt + li * D, ln, A, beta);
            HMM_STAMP(7);
            if (nr > 0)
                warp_store(p.smoothed + ((size_t)b * T + ch0 + r0) * D, tile + (size_t)r0 * D, (int64_t)nr * D);
            warp_store_wait();
            __syncthreads();
            HMM_STAMP(8);
        }
    } else {
        // ===================== Viterbi pass 2: forward sweeps with backpointers, leaf/chunk maps
        uint8_t* bp = smem + p.L.bp;
        uint64_t* maps = reinterpret_cast<uint64_t*>(smem + p.L.maps);
        int32_t* ends = reinterpret_cast<int32_t*>(smem + p.L.ends);
        uint64_t* cmaps = reinterpret_cast<uint64_t*>(smem + p.L.cmaps);
        int32_t* cends = reinterpret_cast<int32_t*>(smem + p.L.cends);
        constexpr int BPB = small_bpb(D);
        const size_t cta_chunk_base = (size_t)(b * G + c) * p.K;
        uint64_t* cmap_ws = reinterpret_cast<uint64_t*>(p.ws + p.ws_cmap) + cta_chunk_base;
        for (int k = 0; do_sweep && k < nchunks; k++) {
            const int64_t ch0 = cta0 + (int64_t)k * p.chunk;
            const int nch = (int)(((ch0 + p.chunk < cta1) ? ch0 + p.chunk : cta1) - ch0);
            const int li = tid * S;
            const int ln = (li < nch) ? ((nch - li < S) ? nch - li : S) : 0;
            const bool t0 = (tb + ch0 + li == 0);
            if (!fused) {
                bool dbad = false;
                leaf_pass(ch0, nch, false, false, dbad);
                tree_down<D, true, false>(tree, NT, carr + k * 2 * D, nullptr);
            }
            float V[D];
#pragma unroll
            for (int d = 0; d < D; d++) V[d] = tree[d * 2 * NT + NT + tid];
            uint64_t f = map_identity(D);
            if (ln > 0) {
                int zi;
                f = vit_sweep<D>(tile + li * D, bp + (size_t)li * BPB, ln, t0, A, pv, V, acc, zi);
                if (zi >= 0 && tb + ch0 + li + zi < zero_t) zero_t = tb + ch0 + li + zi;
                if (ch0 + li + ln == T) {  // this leaf ends the sequence: x*_{T-1} = argmax V (smallest)
                    int xs = 0;
                    for (int d = D - 1; d >= 0; d--)
                        if (V[d] == 0.0f) xs = d;
                    flag[0] = xs;
                }
            }
            HMM_STAMP(5);
            maps[NT + tid] = f;
            if (!fused) {
                // spill this warp's backpointers + leaf maps (re-read by pass 3)
                int r0, nr;
                warp_rows(nch, r0, nr);
                if (nr > 0)
                    warp_store(p.ws + p.ws_bp + (cta_chunk_base + k) * (size_t)p.chunk * BPB + (size_t)r0 * BPB,
                               bp + (size_t)r0 * BPB, ((int64_t)nr * BPB + 3) / 4);
                reinterpret_cast<uint64_t*>(p.ws + p.ws_lmap)[(cta_chunk_base + k) * NT + tid] = f;
                warp_store_wait();
            }
            __syncthreads();
            map_tree_up<D>(maps, NT);
            if (!fused && tid == 0) {
                cmaps[k] = maps[1];
                cmap_ws[k] = maps[1];  // persisted for a split-phase finish call
            }
        }
        if (mode == HMM_MODE_VFINISH) {  // chunk maps from the forward call
            for (int x = tid; x < nchunks; x += NT) cmaps[x] = cmap_ws[x];
        }
        // CTA map
        uint64_t F = 0;
        if (mode == HMM_MODE_FULL || mode == HMM_MODE_VFORWARD || mode == HMM_MODE_VFINISH) {
            if (fused) {
                F = maps[1];
            } else {
                __syncthreads();
                for (int x = tid; x < p.KP; x += NT) maps[p.KP + x] = (x < nchunks) ? cmaps[x] : map_identity(D);
                __syncthreads();
                map_tree_up<D>(maps, p.KP);
                F = maps[1];
            }
        }
        // end state of this CTA = (F_{c+1} o ... o F_{G-1})(x_end), x_end = x*_{T-1} (whole sequence) or the
        // end state of this rank (split phase: resolved from the gathered rank records)
        uint64_t* smaps = reinterpret_cast<uint64_t*>(stage);
        int xs = flag[0];
        if (mode == HMM_MODE_FULL || mode == HMM_MODE_VFORWARD) {
            if (tid == 0) {
                *reinterpret_cast<uint64_t*>(myslot + map_off) = F;
                if (c == G - 1) *reinterpret_cast<int32_t*>(myslot + map_off + 16) = flag[0];
            }
            if (G > 1) group_arrive_wait(arrive2, (uint32_t)G);
            else __syncthreads();
        }
        if (mode == HMM_MODE_VFORWARD) {
            // rank record: {map of the whole rank slice, x* of its last step}
            for (int i = tid; i < G; i += NT)
                smaps[i] = __ldcg(reinterpret_cast<const unsigned long long*>(slots + (size_t)i * p.slot_bytes + map_off));
            __syncthreads();
            if (c == 0 && warp == 0) {
                const uint64_t Fr = warp_compose<D>(smaps, 0, G);
                if (lane == 0) *reinterpret_cast<uint64_t*>(p.rec_out) = Fr;
            }
            if (c == G - 1 && tid == 0) *reinterpret_cast<int32_t*>(p.rec_out + 8) = flag[0];
        }
        if (mode == HMM_MODE_FULL || mode == HMM_MODE_VFINISH) {
            if (G > 1 || mode == HMM_MODE_VFINISH) {
                for (int i = c + 1 + tid; i < G; i += NT) {
                    smaps[i] = __ldcg(reinterpret_cast<const unsigned long long*>(slots + (size_t)i * p.slot_bytes + map_off));
                    if (i == G - 1) flag[3] = __ldcg(reinterpret_cast<const int*>(slots + (size_t)i * p.slot_bytes + map_off + 16));
                }
                if (mode == HMM_MODE_VFINISH && tid == 0) {
                    // x* of the whole sequence (last rank), mapped back through the ranks to our right
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
        }
        const bool do_path = (mode == HMM_MODE_FULL || mode == HMM_MODE_VFINISH);
        const int cta_end = flag[1];
        HMM_STAMP(6);
        if (!do_path) {
        } else if (fused) {
            map_tree_down(maps, ends, NT, cta_end);
        } else {
            // chunk maps are still the leaves of the map tree (KP level)
            map_tree_down(maps, ends, p.KP, cta_end);
            for (int x = tid; x < nchunks; x += NT) cends[x] = ends[p.KP + x];
            __syncthreads();
        }
        // ===================== pass 3: backtrack and write the path
        for (int k = nchunks - 1; do_path && k >= 0; k--) {
            const int64_t ch0 = cta0 + (int64_t)k * p.chunk;
            const int nch = (int)(((ch0 + p.chunk < cta1) ? ch0 + p.chunk : cta1) - ch0);
            const int li = tid * S;
            const int ln = (li < nch) ? ((nch - li < S) ? nch - li : S) : 0;
            if (!fused) {
                const uint8_t* src = p.ws + p.ws_bp + (cta_chunk_base + k) * (size_t)p.chunk * BPB;
                load_floats(reinterpret_cast<float*>(bp), reinterpret_cast<const float*>(src),
                            ((int64_t)nch * BPB + 3) / 4, mbar_aux, aux_phase);
                maps[NT + tid] = __ldcg(reinterpret_cast<const unsigned long long*>(p.ws + p.ws_lmap) +
                                        (cta_chunk_base + k) * NT + tid);
                __syncthreads();
                map_tree_up<D>(maps, NT);
                map_tree_down(maps, ends, NT, cends[k]);
            }
            const int xe = ends[NT + tid];
            int32_t* out = reinterpret_cast<int32_t*>(tile);
            if (ln > 0) vit_backtrack<D>(bp + (size_t)li * BPB, out + li, ln, xe);
            int r0, nr;
            warp_rows(nch, r0, nr);
            __syncwarp();
            if (nr > 0) warp_store(p.path + (size_t)b * T + ch0 + r0, out + r0, nr);
            warp_store_wait();
            __syncthreads();
        }
    }

    // ===================== scalars: log Z / log_prob, info (last CTA of the sequence)
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
        // last CTA: fixed-order sum of the G partials (one per thread, then the block tree)
        __threadfence();
        double v = 0.0;
        for (int x = tid; x < G; x += NT) v += __ldcg(reinterpret_cast<const double*>(slots + (size_t)x * p.slot_bytes + map_off + 8));
        const double tot = block_sum<NT>(v, red);
        if (tid == 0) {
            if (p.scalar_out) p.scalar_out[b] = tot;
            const uint32_t badf = atomicExch(bad_flag, 0u);
            const unsigned long long zc = atomicExch(zero_code, 0ull);
            int32_t inf = 0;
            if (badf) inf = -1;
            else if (zc) inf = (int32_t)((1ull << 62) - zc + 1ull);
            if (p.info) p.info[b] = inf;
            // every CTA has passed every wait of this launch: reset the arrival counters
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
static cudaError_t launch_t(unsigned G, unsigned B, size_t smem, bool coop, const KParams& kp, cudaStream_t stream) {
    auto kern = hmm_small_kernel<D, OP>;
    static size_t configured = 0;  // benign race: idempotent attribute set
    if (configured < smem) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(G, B, 1);
    cfg.blockDim = dim3((unsigned)small_nt(D), 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = coop ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, kp);
}

template <int OP>
static cudaError_t launch_op(int D, unsigned G, unsigned B, size_t smem, bool coop, const KParams& kp,
                             cudaStream_t s) {
    switch (D) {
        case 1: return launch_t<1, OP>(G, B, smem, coop, kp, s);
        case 2: return launch_t<2, OP>(G, B, smem, coop, kp, s);
        case 3: return launch_t<3, OP>(G, B, smem, coop, kp, s);
        case 4: return launch_t<4, OP>(G, B, smem, coop, kp, s);
        case 5: return launch_t<5, OP>(G, B, smem, coop, kp, s);
        case 6: return launch_t<6, OP>(G, B, smem, coop, kp, s);
        case 7: return launch_t<7, OP>(G, B, smem, coop, kp, s);
        case 8: return launch_t<8, OP>(G, B, smem, coop, kp, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_small(int D, int op, unsigned G, unsigned B, size_t smem, bool coop, const KParams& kp,
                         cudaStream_t s) {
    return op == 0 ? launch_op<0>(D, G, B, smem, coop, kp, s) : launch_op<1>(D, G, B, smem, coop, kp, s);
}

}  // namespace hmm
