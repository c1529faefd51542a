// hmm_plan.h — launch plan, shared-memory layout and kernel parameter block shared by the host ABI
// (hmm_abi.cu) and the small-D kernels (hmm_small.cu).
#pragma once
#include <cstddef>
#include <cstdint>

#ifndef __CUDACC__
#define __host__
#define __device__
#endif

namespace hmm {

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~static_cast<size_t>(15); }

// Threads (= leaves) per CTA, floats per tree node, bytes per backpointer entry, per D.
__host__ __device__ constexpr int small_nt(int D) { return D <= 4 ? 256 : 128; }
__host__ __device__ constexpr int small_ne(int D) { return D * D > 2 * D ? D * D : 2 * D; }
__host__ __device__ constexpr int small_bpb(int D) { return D <= 4 ? 2 : 4; }

// Shared-memory carve-up (byte offsets from the dynamic smem base).  RC = steps resident per chunk,
// KP = chunks per CTA rounded to a power of two, G = CTAs per sequence (slot staging).
struct SmemLayout {
    size_t tile, regB, carr, bp, tree, maps, ends, cmaps, cends, stage, misc, total;
};

__host__ __device__ inline size_t small_slot_bytes(int D) { return align16((size_t)D * D * 4) + 32; }

__host__ __device__ inline SmemLayout small_smem_layout(int D, int op, int RC, int KP, int G) {
    const int NT = small_nt(D), NE = small_ne(D);
    const int NPM = NT > KP ? NT : KP;
    const size_t tree_bytes = align16((size_t)2 * NPM * NE * 4);
    const size_t stage_bytes = align16((size_t)G * small_slot_bytes(D));
    SmemLayout L{};
    size_t off = 0;
    L.tile = off;
    off += align16((size_t)RC * D * 4);
    if (op == 0) {
        // regB: filtered staging during the sweeps; before them the trees + the CTA-slot staging
        size_t rb = (size_t)RC * D * 4;
        if (tree_bytes + stage_bytes > rb) rb = tree_bytes + stage_bytes;
        L.regB = off;
        L.tree = off;
        L.stage = off + tree_bytes;
        off += align16(rb);
        L.carr = off;
        off += align16((size_t)KP * 2 * D * 4);
        L.bp = L.maps = L.ends = L.cmaps = L.cends = 0;
    } else {
        L.bp = off;
        off += align16((size_t)RC * small_bpb(D));
        L.tree = off;
        off += tree_bytes;
        L.maps = off;
        off += align16((size_t)2 * NPM * 8);
        L.ends = off;
        off += align16((size_t)2 * NPM * 4);
        L.carr = off;
        off += align16((size_t)KP * 2 * D * 4);
        L.cmaps = off;
        off += align16((size_t)KP * 8);
        L.cends = off;
        off += align16((size_t)KP * 4);
        L.stage = off;
        off += stage_bytes;
        L.regB = 0;
    }
    L.misc = off;  // mbarriers (NT/32 + 1), reduction scratch, CTA carries, flags
    off += 1024 + (size_t)(NT / 32) * 8;
    L.total = align16(off);
    return L;
}

// Work decomposition (DESIGN.md §"Decomposition"):
//   sequence b  ->  G CTAs; CTA c owns steps [c*R, min((c+1)*R, T))
//   CTA range   ->  K chunks of `chunk` steps (K == 1: "fused", the tile stays resident in SMEM)
//   chunk       ->  NT leaves of S consecutive steps, one leaf per thread (S odd: conflict-free SMEM)
struct Plan {
    int D = 0;
    int op = 0;          // 0 smoother, 1 Viterbi
    int64_t T = 0;       // steps per sequence
    int64_t B = 0;       // sequences
    int G = 1;           // CTAs per sequence
    int64_t R = 0;       // steps per CTA (multiple of 8)
    int S = 1;           // steps per leaf (odd)
    int NT = 256;        // threads (= leaves) per CTA
    int chunk = 0;       // steps per chunk (multiple of 8)
    int K = 1;           // max chunks per CTA
    int KP = 1;          // K rounded up to a power of two
    bool fused = true;   // K == 1
    bool coop = false;   // G > 1: grid barrier, cooperative launch required
    size_t smem = 0;     // dynamic shared memory bytes
    // workspace layout (byte offsets)
    size_t ws_sync = 0;      // B * 64 B: barrier/info words per sequence
    size_t ws_slots = 0;     // B * G * slot_bytes: per-CTA roots, maps, partial sums
    size_t slot_bytes = 0;
    size_t ws_chunk = 0;     // B * G * K * chunk_slot: per-chunk roots (non-fused)
    size_t chunk_slot = 0;
    size_t ws_bp = 0;        // Viterbi non-fused: backpointers, B*G*K*chunk*bpb bytes
    size_t ws_lmap = 0;      // Viterbi non-fused: leaf maps, B*G*K*NT*8 bytes
    size_t ws_cmap = 0;      // Viterbi non-fused: chunk maps, B*G*K*8 bytes
    size_t ws_total = 0;
};

struct KParams {
    int64_t T;
    int64_t R;
    int S;
    int chunk;
    int K;
    int KP;
    int fused;
    const float* log_pi;
    const float* log_A;
    const float* log_lik;
    float* filtered;
    float* smoothed;
    int32_t* path;
    double* scalar_out;  // log_likelihood or log_prob, [B]
    int32_t* info;       // [B]
    uint8_t* ws;
    size_t ws_sync, ws_slots, slot_bytes, ws_chunk, chunk_slot, ws_bp, ws_lmap;
    SmemLayout L;
    unsigned long long* timers;  // optional [B*G*16] %globaltimer stamps per CTA phase (profiling only)
    // split-phase distributed execution; mode 0 = whole sequence in one call
    int mode;             // 0 full, 1 reduce, 2 smoother finish, 3 Viterbi forward, 4 Viterbi finish
    int rank, world;
    int64_t t_base;       // global index of local step 0
    const float* agg_all; // [world][agg_stride] rank aggregates (modes 2, 3)
    int agg_stride;       // floats between aggregates
    float* agg_out;       // this rank's aggregate (mode 1)
    const uint8_t* rec_all;  // [world][16] Viterbi rank records {u64 map, i32 x*} (mode 4)
    uint8_t* rec_out;        // this rank's record (mode 3)
    size_t ws_cmap;          // per-chunk Viterbi maps persisted between modes 3 and 4
    // variable-length batches: sequence b = packed rows [offsets[b], offsets[b+1]),
    // 1 <= length <= T (T = the batch's max length); null = every sequence has T rows at b*T
    const int64_t* offsets;
    int64_t pi_stride, A_stride;  // per-sequence models: log_pi + b*pi_stride, log_A + b*A_stride (0: shared)
};


// Sequence b of a (possibly variable-length) batch: its length, clamped to [0, Tmax], and its first row
// in the packed sequence buffers.  `raw` receives the unclamped length (validity is reported in info).
__host__ __device__ __forceinline__ int64_t seq_span(const int64_t* offsets, int64_t Tmax, int64_t b, int64_t& base,
                                                     int64_t& raw) {
    if (!offsets) {
        base = b * Tmax;
        raw = Tmax;
        return Tmax;
    }
    base = offsets[b];
    raw = offsets[b + 1] - base;
    return raw < 0 ? 0 : (raw > Tmax ? Tmax : raw);
}
constexpr int32_t kInfoBadLength = -4;  // HMM_INFO_BAD_LENGTH (hmmscan.h)

// ---------------------------------------------------------------------------- lane streaming
// Long single sequences (DESIGN.md §"Streaming"): lane g = c*NT + tid of the G CTAs owns the
// contiguous steps [g*n, min((g+1)*n, T)), walked in slices of S steps staged by per-lane bulk copies.
__host__ __device__ constexpr int stream_nt(int D) { return D <= 4 ? 256 : 128; }
__host__ __device__ constexpr int stream_s(int D) {
    return D == 1 ? 64 : D == 2 ? 32 : D == 3 ? 20 : D == 4 ? 16 : D == 5 ? 12 : 8;
}
// per-lane SMEM slot: S rows + 16 B (the pad staggers lanes across banks for LDS.128)
__host__ __device__ constexpr int stream_pitch(int D) { return stream_s(D) * D * 4 + 16; }
// bytes of one stored D x D matrix (16-B aligned slot)
__host__ __device__ constexpr int stream_qb(int D) { return (D * D * 4 + 15) & ~15; }

struct StreamLayout {
    size_t ring, qbuf, tab, tree, maps, ends, stage, misc, total;
};
constexpr int kStreamMaxV = 256;  // symbol alphabet of the symbol-input entry points (uint8 y)
__host__ __device__ inline StreamLayout stream_smem_layout(int D, int G) {
    const int NT = stream_nt(D), NE = small_ne(D);
    StreamLayout L{};
    const size_t ring = (size_t)3 * NT * stream_pitch(D);
    L.ring = 0;
    L.tree = 0;  // the trees and the CTA-root staging reuse the ring between the passes
    L.maps = align16((size_t)2 * NT * NE * 4);
    L.ends = L.maps + align16((size_t)2 * NT * 8);
    L.stage = L.ends + align16((size_t)2 * NT * 4);
    size_t u = L.stage + align16((size_t)G * small_slot_bytes(D));
    if (u < ring) u = ring;
    L.qbuf = align16(u);
    L.tab = L.qbuf + (size_t)NT * stream_qb(D);   // symbol table log_B^T [V][D] (symbol inputs)
    L.misc = L.tab + align16((size_t)kStreamMaxV * D * 4);
    L.total = align16(L.misc + 512);
    return L;
}

struct SParams {
    int64_t T;       // steps (local slice in split-phase modes)
    int64_t n;       // steps per lane (multiple of S)
    int K;           // slices per lane = n / S
    const float* log_pi;
    const float* log_A;
    const float* log_lik;
    float* filtered;
    float* smoothed;
    int32_t* path;
    double* scalar_out;
    int32_t* info;
    uint8_t* ws;
    size_t ws_sync, ws_slots, slot_bytes;
    size_t ws_q;     // smoother: [G][K][NT] suffix products of each lane's later slices (QB bytes each)
    size_t ws_lagg;  // [G][NT] lane aggregates (split phase: reduce -> finish / forward)
    size_t ws_bp;    // Viterbi: backpointers by local step (bpb bytes each)
    size_t ws_lmap;  // Viterbi: [G][NT] lane maps (split phase: forward -> finish)
    size_t ws_stats; // smoother statistics: [G][D*D + D] fp64 CTA partials
    double* xi_out;    // [D*D] sum_t xi_t (E-step statistics), or unused
    double* gamma_out; // [D]   sum_t gamma_t
    const uint8_t* y;  // symbol inputs (OP 3/4): y[T] and log_B[D][V]; log_lik rows are gathered on chip
    const float* log_B;
    int V;
    StreamLayout L;
    unsigned long long* timers;
    int mode, rank, world;
    int64_t t_base;
    const float* agg_all;
    int agg_stride;
    float* agg_out;
    const uint8_t* rec_all;
    uint8_t* rec_out;
};

enum { HMM_MODE_FULL = 0, HMM_MODE_REDUCE = 1, HMM_MODE_SFINISH = 2, HMM_MODE_VFORWARD = 3, HMM_MODE_VFINISH = 4 };

}  // namespace hmm
