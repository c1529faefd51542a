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
#include "hmm_small_ops.cuh"

namespace hmm {

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
    int64_t sbase, T_raw;  // first packed row of sequence b, its length (varlen batches: f4)
    const int64_t T = seq_span(p.offsets, p.T, b, sbase, T_raw);
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
    const float* ll_seq = p.log_lik + (size_t)sbase * D;

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
        const float la = __ldg(p.log_A + b * p.A_stride + e);
        A[e] = MP ? la : ex2(la * kLog2e);
    }
#pragma unroll
    for (int d = 0; d < D; d++) {
        const float lp = __ldg(p.log_pi + b * p.pi_stride + d);
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
            copy_root_slots(stage, slots, G, p.slot_bytes, tid, NT);
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
                warp_store(p.filtered + ((size_t)sbase + ch0 + r0) * D, filt + (size_t)r0 * D, (int64_t)nr * D);
            if (tmr && tid == 0) tmr[15] = clock64();
            HMM_STAMP(6);
            if (ln > 0) sp_beta<D>(tile + li * D, filt + li * D, ln, A, beta);
            HMM_STAMP(7);
            if (nr > 0)
                warp_store(p.smoothed + ((size_t)sbase + ch0 + r0) * D, tile + (size_t)r0 * D, (int64_t)nr * D);
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
            if (nr > 0) warp_store(p.path + (size_t)sbase + ch0 + r0, out + r0, nr);
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
            if (T_raw < 1 || T_raw > p.T) inf = kInfoBadLength;
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
    if (cudaError_t e = ensure_smem_optin(reinterpret_cast<const void*>(kern), smem); e != cudaSuccess) return e;
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
