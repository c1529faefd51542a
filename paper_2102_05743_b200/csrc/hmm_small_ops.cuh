// hmm_small_ops.cuh — device building blocks of the small-D (D <= 8) kernels: semiring products,
// SMEM trees, warp reductions, tile movement, leaf folds and the sequential sweeps.  Shared by the
// chunked/fused kernel (hmm_small.cu) and the lane-streaming kernel (hmm_stream.cu).
#pragma once
#include <cfloat>
#include <cstdint>

#include "hmm_device.cuh"

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
// matrix x column vector in either semiring: y(i) = (+)_j M(i,j) (x) v(j), normalised (pow2 / max 0)
// [backward carry; the max-plus form serves Algorithm 5's reversed scan, Prop. 3]
template <int D, bool MP>
__device__ __forceinline__ void mat_vec_sr(const float* M, const float* v, float* y) {
    if constexpr (!MP) {
        mat_vec<D>(M, v, y);
    } else {
#pragma unroll
        for (int i = 0; i < D; i++) {
            float s[D];
#pragma unroll
            for (int j = 0; j < D; j++) s[j] = M[i * D + j] + v[j];
            y[i] = vmax<D>(s);
        }
        const float m = vmax<D>(y);
        if (m > neg_inf()) {
#pragma unroll
            for (int i = 0; i < D; i++) y[i] -= m;
        }
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
                    if (SUF) {
#pragma unroll
                        for (int j = 0; j < D; j++) sc[j] = tree[(d * D + j) * NN + 2 * x + 1] + suf[j];
                        sl = vmax<D>(sc);
                    }
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
                    if (SUF && ms > neg_inf()) sl -= ms;
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
                    mat_vec_sr<D, MP>(Rm, suf, sufL);
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
// D = 4 leaf: two chains (rows [0, h) and [h, n), combined at the end: 2x ILP on the latency-bound fold)
// of packed column-pair steps, P <- P psi_t = (P A) diag(l_t) as FMUL2 / FFMA2 with the broadcast P(r,k);
// the exact power-of-two renormalisation is folded into the next step's ex2 argument (d = 127 - E(max)),
// so it costs no multiplies.  The l rows written back for the sweeps then carry that factor 2^d: the
// sweeps are scale-free except log Z, from which the written factors' sum (an exact integer times ln 2)
// is removed here.
__device__ __forceinline__ void sp_leaf4_step(const float* row, float* wrow, bool start, bool t0, const float2* A2,
                                              const float* pi, float2* P2, float& d, float& dsum, double& msum,
                                              bool acc_m) {
    float v[4];
    ld_row<4>(row, v);
    const float mr = fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3]));
    if (acc_m && mr > neg_inf()) msum += (double)mr;
    const float m = fmaxf(mr, -1e30f);  // all -inf (impossible step): l = 0
    const float c = fmaf(-m, kLog2e, d);
    float l[4];
#pragma unroll
    for (int j = 0; j < 4; j++) l[j] = ex2(fmaf(v[j], kLog2e, c));
    if (wrow) {
        st_row<4>(wrow, l);
        dsum += d;
    }
    const float2 l2[2] = {make_float2(l[0], l[1]), make_float2(l[2], l[3])};
    if (start) {
#pragma unroll
        for (int r = 0; r < 4; r++)
#pragma unroll
            for (int jj = 0; jj < 2; jj++)
                P2[r * 2 + jj] = t0 ? __fmul2_rn(make_float2(pi[2 * jj], pi[2 * jj + 1]), l2[jj])
                                    : __fmul2_rn(A2[r * 2 + jj], l2[jj]);
    } else {
        float2 R2[8];
#pragma unroll
        for (int k = 0; k < 4; k++)
#pragma unroll
            for (int jj = 0; jj < 2; jj++) R2[k * 2 + jj] = __fmul2_rn(A2[k * 2 + jj], l2[jj]);
        float2 Pn[8];
#pragma unroll
        for (int r = 0; r < 4; r++) {
            const float p0 = P2[r * 2].x, p1 = P2[r * 2].y, p2 = P2[r * 2 + 1].x, p3 = P2[r * 2 + 1].y;
#pragma unroll
            for (int jj = 0; jj < 2; jj++) {
                float2 acc = __fmul2_rn(make_float2(p0, p0), R2[jj]);
                acc = __ffma2_rn(make_float2(p1, p1), R2[2 + jj], acc);
                acc = __ffma2_rn(make_float2(p2, p2), R2[4 + jj], acc);
                acc = __ffma2_rn(make_float2(p3, p3), R2[6 + jj], acc);
                Pn[r * 2 + jj] = acc;
            }
        }
#pragma unroll
        for (int e = 0; e < 8; e++) P2[e] = Pn[e];
    }
    float mx[8];
#pragma unroll
    for (int e = 0; e < 8; e++) mx[e] = fmaxf(P2[e].x, P2[e].y);
    d = exp_offset(vmax2_tree<8>(mx));
}

template <int D>
__device__ __forceinline__ void sp_leaf(float* rows, int n, bool t0, const float* A, const float* pi, float* P,
                                        double& msum, bool write_l, bool acc_m, bool& bad) {
    if constexpr (D == 4) {
        float2 A2[8];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            A2[k * 2] = make_float2(A[k * 4], A[k * 4 + 1]);
            A2[k * 2 + 1] = make_float2(A[k * 4 + 2], A[k * 4 + 3]);
        }
        const int h = (n + 1) / 2;  // chain X: rows [0, h); chain Y: rows [h, n)
        float2 X2[8], Y2[8];
        float dx = 0.0f, dy = 0.0f, dsum = 0.0f;
        double mx = 0.0, my = 0.0;
        for (int q = 0; q < h; q++) {
            sp_leaf4_step(rows + q * 4, write_l ? rows + q * 4 : nullptr, q == 0, t0 && q == 0, A2, pi, X2, dx, dsum,
                          mx, acc_m);
            if (h + q < n)
                sp_leaf4_step(rows + (h + q) * 4, write_l ? rows + (h + q) * 4 : nullptr, q == 0, false, A2, pi, Y2,
                              dy, dsum, my, acc_m);
        }
        msum += mx + my - (double)dsum * (double)kLn2;
        float X[16], Y[16];
#pragma unroll
        for (int e = 0; e < 8; e++) {
            X[2 * e] = X2[e].x; X[2 * e + 1] = X2[e].y;
            Y[2 * e] = Y2[e].x; Y[2 * e + 1] = Y2[e].y;
        }
        if (n > h) mat_op<4, false>(X, Y, P);  // (renormalised by an exact power of two)
        else {
            const float s = pow2_inv(vmax<16>(X));
#pragma unroll
            for (int e = 0; e < 16; e++) P[e] = X[e] * s;
        }
        const float chk = vsum<16>(P);  // a NaN or +inf input anywhere in the leaf leaves a NaN here
        bad |= (chk != chk);
        return;
    }
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
            float sc[D];
#pragma unroll
            for (int k = 0; k < D; k++) sc[k] = V[k] + (first ? LP[j] : LA[k * D + j]);
            // max by a 2-input tree (short V critical path); argmax = smallest index attaining it
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

}  // namespace hmm
