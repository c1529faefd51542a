// hmm_abi.cu — extern "C" entry points of libhmmscan.so (declared in include/hmmscan.h):
// argument validation, launch planning (work decomposition, shared memory, workspace layout) and
// dispatch to the sm_100a kernels.  No compute happens on the host.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>

#include "../../include/hmmscan.h"
#include "hmm_large.h"
#include "hmm_plan.h"

namespace hmm {
cudaError_t launch_small(int D, int op, unsigned G, unsigned B, size_t smem, bool coop, const KParams& kp,
                         cudaStream_t s);
cudaError_t launch_large(int DP, int op, const LgParams& p, cudaStream_t s);
cudaError_t launch_stream(int D, int op, unsigned G, const SParams& sp, cudaStream_t s);
int large_leaves_per_block(int DP);
size_t variants_workspace_size(int op, int D, int64_t T, int64_t B);
cudaError_t launch_batchseq(int DP, int op, bool bidir, const BSParams& p, cudaStream_t s);
int64_t bs2_beta_rows(int64_t Tmax);
size_t bs_smem(int DP, int op, bool bidir);
}

using hmm::Plan;

namespace hmm {
cudaError_t ensure_smem_optin(const void* func, size_t smem) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> applied;  // (device, kernel) -> bytes set
    int dev = 0;
    if (cudaError_t e = cudaGetDevice(&dev); e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    size_t& have = applied[{dev, func}];
    if (have >= smem) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) have = smem;
    return e;
}
}  // namespace hmm

namespace {

struct DevInfo {
    int sms = 0;
    int smem_optin = 0;
};

constexpr int kMaxDevices = 64;
DevInfo g_dev[kMaxDevices];
std::once_flag g_dev_once[kMaxDevices];

bool dev_info(DevInfo& out) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return false;
    std::call_once(g_dev_once[dev], [dev]() {
        cudaDeviceGetAttribute(&g_dev[dev].sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&g_dev[dev].smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    });
    out = g_dev[dev];
    return out.sms > 0;
}

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
int64_t round_up(int64_t a, int64_t b) { return cdiv(a, b) * b; }
int pow2_ceil(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

// Work decomposition for the small-D kernels (see hmm_plan.h and DESIGN.md §"Decomposition").
bool make_plan(int D, int op, int64_t T, int64_t B, Plan& P, bool chunked = false, bool one_cta = false) {
    DevInfo di;
    if (!dev_info(di)) return false;
    P = Plan{};
    P.D = D; P.op = op; P.T = T; P.B = B;
    P.NT = hmm::small_nt(D);
    const int NT = P.NT;
    const size_t smax = (size_t)di.smem_optin;
    int64_t G;
    if (B >= di.sms || one_cta) {  // (variable-length batches: one CTA per sequence, f4)
        G = 1;
    } else {
        G = di.sms / B;
        const int64_t gmax = cdiv(T, (int64_t)NT * 8);  // >= ~8 steps per thread
        if (G > gmax) G = gmax;
        if (G < 1) G = 1;
    }
    int64_t R = round_up(cdiv(T, G), 8);
    G = cdiv(T, R);
    P.G = (int)G;
    P.R = R;
    // fused: the whole CTA range stays resident in shared memory
    hmm::SmemLayout Lf = hmm::small_smem_layout(D, op, (int)std::min<int64_t>(R, 1 << 30), 1, (int)G);
    if (!chunked && R <= (1 << 24) && Lf.total <= smax) {
        int S = (int)cdiv(R, NT);
        if ((S & 1) == 0) S += 1;
        P.S = S;
        P.chunk = (int)R;
        P.K = 1;
        P.KP = 1;
        P.fused = true;
        P.smem = Lf.total;
    } else {
        int S = 25;
        for (;;) {
            const int chunk = NT * S;
            const int K = (int)cdiv(R, chunk);
            const int KP = pow2_ceil(K);
            hmm::SmemLayout L = hmm::small_smem_layout(D, op, chunk, KP, (int)G);
            if (chunked && (int64_t)chunk > R && S > 3) {  // split-phase: keep chunks no longer than the range
                S -= 2;
                continue;
            }
            if (L.total <= smax && KP <= 1024) {
                P.S = S; P.chunk = chunk; P.K = K; P.KP = KP; P.smem = L.total;
                break;
            }
            if (KP > 1024) S += 2; else S -= 2;
            if (S < 3 || S > 255) return false;
        }
        P.fused = false;
    }
    P.coop = P.G > 1;
    // workspace
    size_t off = 0;
    P.ws_sync = off;
    off += hmm::align16((size_t)B * 64);
    off = (off + 255) & ~(size_t)255;
    P.slot_bytes = hmm::small_slot_bytes(D);
    P.ws_slots = off;
    off += (size_t)B * P.G * P.slot_bytes;
    off = (off + 255) & ~(size_t)255;
    P.chunk_slot = hmm::align16((size_t)D * D * 4);
    P.ws_chunk = off;
    if (!P.fused) off += (size_t)B * P.G * P.K * P.chunk_slot;
    off = (off + 255) & ~(size_t)255;
    P.ws_bp = off;
    if (op == 1 && !P.fused) off += (size_t)B * P.G * P.K * (size_t)P.chunk * hmm::small_bpb(D);
    off = (off + 255) & ~(size_t)255;
    P.ws_lmap = off;
    if (op == 1 && !P.fused) off += (size_t)B * P.G * P.K * (size_t)NT * 8;
    off = (off + 255) & ~(size_t)255;
    P.ws_cmap = off;
    if (op == 1 && !P.fused) off += (size_t)B * P.G * P.K * 8;
    off = (off + 255) & ~(size_t)255;
    P.ws_total = off;
    return true;
}

thread_local int t_force_path = 0;  // hmm_debug_force_path

// Lane-streaming plan (hmm_stream.cu): G CTAs of NT lanes, n steps per lane (a multiple of the slice
// length S), K = n / S slices per lane.
struct StPlan {
    int G = 1;
    int64_t n = 0;
    int K = 0;
    size_t smem = 0;
    size_t ws_sync, ws_slots, slot_bytes, ws_q, ws_lagg, ws_bp, ws_lmap, ws_stats, ws_total;
};

bool make_stream_plan(int D, int op, int64_t T, StPlan& P) {
    DevInfo di;
    if (!dev_info(di) || D < 1 || D > 8) return false;
    P = StPlan{};
    const int NT = hmm::stream_nt(D), S = hmm::stream_s(D);
    int64_t G = cdiv(T, (int64_t)NT * S);
    if (G > di.sms) G = di.sms;
    int64_t n = round_up(cdiv(T, G * NT), S);
    G = cdiv(T, n * NT);
    if (G < 1) G = 1;
    P.G = (int)G;
    P.n = n;
    P.K = (int)(n / S);
    hmm::StreamLayout L = hmm::stream_smem_layout(D, P.G);
    if (L.total > (size_t)di.smem_optin) return false;
    P.smem = L.total;
    const size_t lanes = (size_t)P.G * NT, QB = hmm::stream_qb(D);
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = (off + bytes + 255) & ~(size_t)255; return o; };
    P.ws_sync = take(64);
    P.slot_bytes = hmm::small_slot_bytes(D);
    P.ws_slots = take((size_t)P.G * P.slot_bytes);
    P.ws_q = take(op != 1 ? lanes * P.K * QB : 0);
    P.ws_lagg = take(lanes * QB);
    P.ws_bp = take(op == 1 ? (size_t)(T + S) * hmm::small_bpb(D) + 16 : 0);
    P.ws_lmap = take(op == 1 ? lanes * 8 : 0);
    P.ws_stats = take(op == 2 ? (size_t)P.G * (D * D + D) * 8 : 0);
    P.ws_total = off;
    return true;
}

// Long single sequences whose CTA ranges do not fit in shared memory take the streaming kernel
// (as do all split-phase calls); it needs 16-B aligned sequence buffers for its bulk copies.
bool use_stream(int D, int64_t T, int64_t B, bool dist) {
    if (D > 8 || B != 1) return false;
    if (t_force_path == 1) return true;
    if (t_force_path == 2) return false;
    if (dist) return true;
    Plan P;
    if (!make_plan(D, 0, T, B, P)) return true;
    return !P.fused;
}
bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Batch-parallel plan (hmm_batchseq.cu) for 9 <= D <= 32: one lane group per sequence running the
// element recursions; chosen when the batch is large enough that the scan's D^3 element products cost
// more than the recursions' per-step latency.  hmm_debug_force_path: 4 forces it,
// 5 forbids it.
int bs_dp(int D) { return D <= 16 ? 16 : (D <= 32 ? 32 : 0); }
// The plan's time is T x (per-step latency of the recursion) until the batch saturates the issue slots;
// the scan's is proportional to B T D^3.  Measured crossover with the bidirectional variant
// (tools/batchseq_crossover.py, T = 4096, profiles/r2/bidir/crossover.txt; T cancels): DP = 16 smoother
// B ~ 380, Viterbi ~ 300; DP = 32 below B = 128 for both.
bool use_batchseq(int D, int op, int64_t B) {
    const int DP = bs_dp(D);
    if (D <= 8 || DP == 0) return false;
    if (t_force_path == 4 || t_force_path == 6) return true;
    if (t_force_path == 5) return false;
    const int64_t bmin = DP == 16 ? (op == 0 ? 384 : 320) : 64;
    return B >= bmin;
}
// Bidirectional variant (hmm_batchseq.cu): the forward and backward recursions run at the same time from
// the two ends, halving the per-sequence latency; it holds as many sequences per SM as the one-warp plan
// (DP = 16) or more (DP = 32), so it is the batch-parallel plan at every B (profiles/r2/bidir:
// D = 16, B = 2048: 1.95 vs 3.33 ms; D = 32, B = 1024: 2.46 vs 4.27 ms).  hmm_debug_force_path 6 forces
// the one-warp plan (tests).
bool bs_bidir(int D, int op, int64_t B) {
    (void)D; (void)op; (void)B;
    return t_force_path != 6;
}
size_t bs_workspace(int op, int D, int64_t T, int64_t B) {
    if (op == 1) return ((size_t)B * T * bs_dp(D) + 255) & ~(size_t)255;
    return ((size_t)B * (size_t)hmm::bs2_beta_rows(T) * (size_t)D * 4 + 511) & ~(size_t)255;
}
hmm_status_t run_batchseq(int op, int D, int64_t T, int64_t B, const int64_t* offsets, int64_t pis, int64_t As,
                          const float* log_pi, const float* log_A, const float* log_lik, float* filtered,
                          float* smoothed, int32_t* path, double* scalar, int32_t* info, void* ws, size_t ws_bytes,
                          void* stream) {
    if (!ws || ws_bytes < bs_workspace(op, D, T, B) || (reinterpret_cast<uintptr_t>(ws) & 255u)) return HMM_ERR_WORKSPACE;
    hmm::BSParams bp;
    std::memset(&bp, 0, sizeof(bp));
    bp.T = T; bp.B = B; bp.D = D;
    bp.log_pi = log_pi; bp.log_A = log_A; bp.log_lik = log_lik;
    bp.filtered = filtered; bp.smoothed = smoothed; bp.path = path; bp.scalar_out = scalar; bp.info = info;
    bp.bp = static_cast<uint8_t*>(ws);
    bp.sbeta = static_cast<float*>(ws);
    bp.s_rows = hmm::bs2_beta_rows(T);
    bp.offsets = offsets; bp.pi_stride = pis; bp.A_stride = As;
    const cudaError_t e = hmm::launch_batchseq(bs_dp(D), op, bs_bidir(D, op, B), bp, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? HMM_SUCCESS : HMM_ERR_CUDA;
}

// Profiling hook (hmm_debug_set_timers): per-thread, not used unless set.
thread_local unsigned long long* t_timers = nullptr;

// Large-D plan (9 <= D <= 64): DP = padded state count; leaves of SL steps, NLB leaves per CTA.
struct LgPlan {
    int DP = 0;
    bool tc = false;  // sum-product leaf products on the tensor cores (DP = 64)
    int64_t SL = 0, NL = 0, NB = 0;
    int64_t KG = 0, NG = 1;  // two-level carry: KG block roots per group, NG groups (NG = 1: one level)
    size_t o_sync, o_leaf, o_groot, o_bpre, o_bsuf, o_part, o_bp, o_lmap, o_bmap, o_bend, o_xstar, o_lik;
    size_t o_gprod, o_gpre, o_gsuf, o_rcar, total;
};

bool make_large_plan(int D, int op, int64_t T, int64_t B, LgPlan& P, bool allow_tc = true) {
    DevInfo di;
    if (!dev_info(di)) return false;
    P.DP = D <= 16 ? 16 : (D <= 32 ? 32 : 64);
    const int NLB = hmm::large_leaves_per_block(P.DP);
    P.tc = (P.DP == 64 && op == 0 && t_force_path != 3 && allow_tc);
    // enough leaves for ~2 waves of 8-warp CTAs, leaves between 16 and 512 steps; the tensor-core
    // leaf kernel runs 2 leaf pairs per SM, so it wants ~4 leaves per SM
    // (tensor-core leaves: 2 leaf pairs per SM per wave; 2 waves so the sweep kernel, NLB leaves
    // per CTA, still covers every SM)
    // (DP = 64 on CUDA cores: one 256-thread CTA per SM (214 registers), so two waves of blocks buy no
    // balance and only double the serial block-root chains of the carry / resolve kernels: one wave)
    const int64_t target = P.tc ? (int64_t)di.sms * 8 : (int64_t)di.sms * (P.DP == 64 ? 1 : 2) * NLB;
    int64_t SL = cdiv(T * B, target);
    // many sequences (one block each): fill every block's NLB leaf slots -- the leaf chains are
    // latency-bound, so idle slots cost throughput directly
    if (!P.tc && B >= di.sms) SL = cdiv(T, NLB);
    if (SL < 16) SL = 16;
    if (SL > (P.tc ? 2048 : 512)) SL = P.tc ? 2048 : 512;
    if (SL > T) SL = T;
    P.SL = SL;
    P.NL = cdiv(T, SL);
    P.NB = cdiv(P.NL, NLB);
    // The block-root carry chain is serial (~1 us per root at DP = 64): beyond 24 roots it runs in two
    // levels, ~sqrt(NB / 2) roots per group (hmm_large.cu lg_group_kernel).
    P.KG = P.NB;
    P.NG = 1;
    if (P.NB > 24) {  // group product ~2.5 us per root, chain steps ~0.9 us: KG ~ sqrt(NB / 2)
        int64_t kg = 6;
        while (2 * kg * kg < P.NB) kg++;
        P.KG = kg;
        P.NG = cdiv(P.NB, kg);
    }
    const size_t DP2 = (size_t)P.DP * P.DP;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = (off + bytes + 255) & ~(size_t)255; return o; };
    P.o_sync = take((size_t)B * 64);
    P.o_leaf = take((size_t)B * P.NL * DP2 * 4);
    P.o_groot = take((size_t)B * P.NB * DP2 * 4);
    P.o_bpre = take((size_t)B * P.NB * P.DP * 4);
    P.o_bsuf = take((size_t)B * P.NB * P.DP * 4);
    P.o_part = take((size_t)B * P.NL * 8);
    P.o_bp = take(op == 1 ? (size_t)B * T * P.DP : 0);
    P.o_lmap = take(op == 1 ? (size_t)B * P.NL * P.DP : 0);
    P.o_bmap = take(op == 1 ? (size_t)B * P.NB * P.DP : 0);
    P.o_bend = take(op == 1 ? (size_t)B * P.NB * 4 : 0);
    P.o_xstar = take((size_t)B * 4);
    P.o_lik = take(P.tc ? (size_t)B * T * 64 * 4 : 0);
    P.o_gprod = take(P.NG > 1 ? (size_t)B * P.NG * DP2 * 4 : 0);
    P.o_gpre = take(P.NG > 1 ? (size_t)B * P.NG * P.DP * 4 : 0);
    P.o_gsuf = take(P.NG > 1 ? (size_t)B * P.NG * P.DP * 4 : 0);
    P.o_rcar = take((size_t)2 * P.DP * 4);  // split-phase rank carries
    P.total = off;
    return true;
}

bool al4(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 3u) == 0; }
bool al8(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 7u) == 0; }

struct DistArgs {
    int mode = 0, rank = 0, world = 1;
    int64_t t_base = 0;
    const float* agg_all = nullptr;
    float* agg_out = nullptr;
    const uint8_t* rec_all = nullptr;
    uint8_t* rec_out = nullptr;
};

hmm_status_t run(int op, int D, int64_t T, int64_t B, const float* log_pi, const float* log_A, const float* log_lik,
                 float* filtered, float* smoothed, int32_t* path, double* scalar, int32_t* info, void* ws,
                 size_t ws_bytes, void* stream, const DistArgs& da = DistArgs()) {
    if (D < 1 || T < 1 || B < 1 || B > 65535) return HMM_ERR_INVALID_VALUE;
    if (D > HMM_MAX_D) return HMM_ERR_UNSUPPORTED;
    // split phase at D > 8 (one sequence): smoother reduce / finish, Viterbi reduce / forward / finish
    if (D > 8 && da.mode != hmm::HMM_MODE_FULL &&
        (B != 1 || (op == 0 && da.mode != hmm::HMM_MODE_REDUCE && da.mode != hmm::HMM_MODE_SFINISH) ||
         (op == 1 && da.mode != hmm::HMM_MODE_REDUCE && da.mode != hmm::HMM_MODE_VFORWARD &&
          da.mode != hmm::HMM_MODE_VFINISH)))
        return HMM_ERR_UNSUPPORTED;
    if (D > 8) {
        const bool ldist = da.mode != hmm::HMM_MODE_FULL;
        const bool lreduce = da.mode == hmm::HMM_MODE_REDUCE;
        const bool vfwd = da.mode == hmm::HMM_MODE_VFORWARD, vfin = da.mode == hmm::HMM_MODE_VFINISH;
        const bool need_sc = !lreduce && !vfin;
        if (!log_pi || !log_A || !log_lik || (need_sc && !scalar) || !info) return HMM_ERR_INVALID_VALUE;
        if (op == 0 && !lreduce && !smoothed) return HMM_ERR_INVALID_VALUE;
        if (op == 1 && (da.mode == hmm::HMM_MODE_FULL || vfin) && !path) return HMM_ERR_INVALID_VALUE;
        if (op == 0 && !lreduce && !filtered) return HMM_ERR_UNSUPPORTED;  // large-D smoother stages alpha in `filtered`
        if (!al4(log_pi) || !al4(log_A) || !al4(log_lik) || (scalar && !al8(scalar)) || !al4(info))
            return HMM_ERR_INVALID_VALUE;
        if (ldist && (da.world < 1 || da.rank < 0 || da.rank >= da.world || da.t_base < 0 ||
                      (lreduce && !da.agg_out) || ((da.mode == hmm::HMM_MODE_SFINISH || vfwd) && !da.agg_all) ||
                      (vfwd && !da.rec_out) || (vfin && !da.rec_all)))
            return HMM_ERR_INVALID_VALUE;
        if (!ldist && use_batchseq(D, op, B))
            return run_batchseq(op, D, T, B, nullptr, 0, 0, log_pi, log_A, log_lik, filtered, smoothed, path, scalar,
                                info, ws, ws_bytes, stream);
        LgPlan G;
        if (!make_large_plan(D, op, T, B, G)) return HMM_ERR_UNSUPPORTED;
        if (!ws || ws_bytes < G.total || (reinterpret_cast<uintptr_t>(ws) & 255u)) return HMM_ERR_WORKSPACE;
        uint8_t* w = static_cast<uint8_t*>(ws);
        hmm::LgParams lp;
        std::memset(&lp, 0, sizeof(lp));
        lp.T = T; lp.B = B; lp.D = D; lp.SL = G.SL; lp.NL = G.NL; lp.NB = G.NB;
        lp.log_pi = log_pi; lp.log_A = log_A; lp.log_lik = log_lik;
        lp.filtered = filtered; lp.smoothed = smoothed; lp.path = path; lp.scalar_out = scalar; lp.info = info;
        lp.ws_sync = w + G.o_sync;
        lp.leafagg = reinterpret_cast<float*>(w + G.o_leaf);
        lp.groot = reinterpret_cast<float*>(w + G.o_groot);
        lp.bpre = reinterpret_cast<float*>(w + G.o_bpre);
        lp.bsuf = reinterpret_cast<float*>(w + G.o_bsuf);
        lp.partial = reinterpret_cast<double*>(w + G.o_part);
        lp.bp = w + G.o_bp;
        lp.lmap = w + G.o_lmap;
        lp.bmap = w + G.o_bmap;
        lp.bend = reinterpret_cast<int32_t*>(w + G.o_bend);
        lp.xstar = reinterpret_cast<int32_t*>(w + G.o_xstar);
        lp.KG = G.KG; lp.NG = G.NG;
        lp.gprod = reinterpret_cast<float*>(w + G.o_gprod);
        lp.gpre = reinterpret_cast<float*>(w + G.o_gpre);
        lp.gsuf = reinterpret_cast<float*>(w + G.o_gsuf);
        lp.rcar = reinterpret_cast<float*>(w + G.o_rcar);
        lp.mode = da.mode; lp.t_base = da.t_base; lp.rank = da.rank; lp.world = da.world;
        lp.agg_all = da.agg_all; lp.agg_out = da.agg_out;
        lp.rec_out = da.rec_out; lp.rec_all = da.rec_all; lp.rec_bytes = (int)hmm_dist_record_bytes_d(D);
        lp.tc = G.tc ? 1 : 0;
        lp.lik = reinterpret_cast<float*>(w + G.o_lik);
        cudaError_t e = hmm::launch_large(G.DP, op, lp, static_cast<cudaStream_t>(stream));
        return e == cudaSuccess ? HMM_SUCCESS : HMM_ERR_CUDA;
    }
    const bool dist = da.mode != hmm::HMM_MODE_FULL;
    const bool need_scalar = !dist || da.mode == hmm::HMM_MODE_SFINISH || da.mode == hmm::HMM_MODE_VFORWARD;
    if (!log_pi || !log_A || !log_lik || !info || (need_scalar && !scalar)) return HMM_ERR_INVALID_VALUE;
    if (op == 0 && (da.mode == hmm::HMM_MODE_FULL || da.mode == hmm::HMM_MODE_SFINISH) && !smoothed)
        return HMM_ERR_INVALID_VALUE;
    if (op == 1 && (da.mode == hmm::HMM_MODE_FULL || da.mode == hmm::HMM_MODE_VFINISH) && !path)
        return HMM_ERR_INVALID_VALUE;
    if (!al4(log_pi) || !al4(log_A) || !al4(log_lik) || (scalar && !al8(scalar)) || !al4(info))
        return HMM_ERR_INVALID_VALUE;
    if ((filtered && !al4(filtered)) || (smoothed && !al4(smoothed)) || (path && !al4(path)))
        return HMM_ERR_INVALID_VALUE;
    if (dist && (D > 8 || B != 1 || da.world < 1 || da.rank < 0 || da.rank >= da.world || da.t_base < 0))
        return D > 8 ? HMM_ERR_UNSUPPORTED : HMM_ERR_INVALID_VALUE;
    // The decomposition: the lane-streaming kernel needs 16-B aligned sequence buffers.  Outside the split
    // phase a misaligned buffer just selects the resident/chunked kernel.  The split-phase calls of one
    // rank must all run the same kernel (the finish/forward calls read the workspace layout the reduce
    // call wrote), so there the choice depends on log_lik alone and misaligned outputs are an error.
    const bool out16 = (!filtered || al16(filtered)) && (!smoothed || al16(smoothed)) && (!path || al16(path));
    bool stream_path = use_stream(D, T, B, dist) && al16(log_lik);
    if (stream_path && !out16) {
        if (dist) return HMM_ERR_INVALID_VALUE;
        stream_path = false;
    }
    if (stream_path) {
        StPlan SP;
        if (!make_stream_plan(D, op, T, SP)) return HMM_ERR_UNSUPPORTED;
        if (!ws || ws_bytes < SP.ws_total || (reinterpret_cast<uintptr_t>(ws) & 255u)) return HMM_ERR_WORKSPACE;
        hmm::SParams sp;
        std::memset(&sp, 0, sizeof(sp));
        sp.T = T; sp.n = SP.n; sp.K = SP.K;
        sp.log_pi = log_pi; sp.log_A = log_A; sp.log_lik = log_lik;
        sp.filtered = filtered; sp.smoothed = smoothed; sp.path = path; sp.scalar_out = scalar; sp.info = info;
        sp.ws = static_cast<uint8_t*>(ws);
        sp.ws_sync = SP.ws_sync; sp.ws_slots = SP.ws_slots; sp.slot_bytes = SP.slot_bytes; sp.ws_q = SP.ws_q;
        sp.ws_lagg = SP.ws_lagg; sp.ws_bp = SP.ws_bp; sp.ws_lmap = SP.ws_lmap;
        sp.L = hmm::stream_smem_layout(D, SP.G);
        sp.timers = t_timers;
        sp.mode = da.mode; sp.rank = da.rank; sp.world = da.world; sp.t_base = da.t_base;
        sp.agg_all = da.agg_all; sp.agg_stride = (int)(hmm::align16((size_t)D * D * 4) / 4);
        sp.agg_out = da.agg_out; sp.rec_all = da.rec_all; sp.rec_out = da.rec_out;
        cudaError_t e = hmm::launch_stream(D, op, (unsigned)SP.G, sp, static_cast<cudaStream_t>(stream));
        return e == cudaSuccess ? HMM_SUCCESS : HMM_ERR_CUDA;
    }
    Plan P;
    if (!make_plan(D, op, T, B, P, dist)) return HMM_ERR_UNSUPPORTED;
    if (!ws || ws_bytes < P.ws_total || (reinterpret_cast<uintptr_t>(ws) & 255u)) return HMM_ERR_WORKSPACE;
    hmm::KParams kp;
    std::memset(&kp, 0, sizeof(kp));
    kp.T = T; kp.R = P.R; kp.S = P.S; kp.chunk = P.chunk; kp.K = P.K; kp.KP = P.KP; kp.fused = P.fused ? 1 : 0;
    kp.log_pi = log_pi; kp.log_A = log_A; kp.log_lik = log_lik;
    kp.filtered = filtered; kp.smoothed = smoothed; kp.path = path; kp.scalar_out = scalar; kp.info = info;
    kp.ws = static_cast<uint8_t*>(ws);
    kp.ws_sync = P.ws_sync; kp.ws_slots = P.ws_slots; kp.slot_bytes = P.slot_bytes;
    kp.ws_chunk = P.ws_chunk; kp.chunk_slot = P.chunk_slot; kp.ws_bp = P.ws_bp; kp.ws_lmap = P.ws_lmap;
    kp.L = hmm::small_smem_layout(D, op, P.chunk, P.KP, P.G);
    kp.timers = t_timers;
    kp.ws_cmap = P.ws_cmap;
    kp.mode = da.mode; kp.rank = da.rank; kp.world = da.world; kp.t_base = da.t_base;
    kp.agg_all = da.agg_all; kp.agg_stride = (int)(hmm::align16((size_t)D * D * 4) / 4);
    kp.agg_out = da.agg_out; kp.rec_all = da.rec_all; kp.rec_out = da.rec_out;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = hmm::launch_small(D, op, (unsigned)P.G, (unsigned)P.B, P.smem, P.coop, kp, s);
    return e == cudaSuccess ? HMM_SUCCESS : HMM_ERR_CUDA;
}

// Smoother + Baum-Welch E-step statistics: lane-streaming kernel only (D <= 8, one sequence).
hmm_status_t run_stats(int D, int64_t T, const float* log_pi, const float* log_A, const float* log_lik,
                       float* filtered, float* smoothed, double* log_likelihood, double* xi_sum, double* gamma_sum,
                       int32_t* info, void* ws, size_t ws_bytes, void* stream) {
    if (D < 1 || T < 1) return HMM_ERR_INVALID_VALUE;
    if (D > 8) return HMM_ERR_UNSUPPORTED;
    if (!log_pi || !log_A || !log_lik || !log_likelihood || !xi_sum || !gamma_sum || !info) return HMM_ERR_INVALID_VALUE;
    if (!al4(log_pi) || !al4(log_A) || !al8(log_likelihood) || !al8(xi_sum) || !al8(gamma_sum) || !al4(info))
        return HMM_ERR_INVALID_VALUE;
    if (!al16(log_lik) || (filtered && !al16(filtered)) || (smoothed && !al16(smoothed))) return HMM_ERR_INVALID_VALUE;
    StPlan SP;
    if (!make_stream_plan(D, 2, T, SP)) return HMM_ERR_UNSUPPORTED;
    if (!ws || ws_bytes < SP.ws_total || (reinterpret_cast<uintptr_t>(ws) & 255u)) return HMM_ERR_WORKSPACE;
    hmm::SParams sp;
    std::memset(&sp, 0, sizeof(sp));
    sp.T = T; sp.n = SP.n; sp.K = SP.K;
    sp.log_pi = log_pi; sp.log_A = log_A; sp.log_lik = log_lik;
    sp.filtered = filtered; sp.smoothed = smoothed; sp.scalar_out = log_likelihood; sp.info = info;
    sp.ws = static_cast<uint8_t*>(ws);
    sp.ws_sync = SP.ws_sync; sp.ws_slots = SP.ws_slots; sp.slot_bytes = SP.slot_bytes; sp.ws_q = SP.ws_q;
    sp.ws_lagg = SP.ws_lagg; sp.ws_stats = SP.ws_stats;
    sp.xi_out = xi_sum; sp.gamma_out = gamma_sum;
    sp.L = hmm::stream_smem_layout(D, SP.G);
    sp.timers = t_timers;
    sp.mode = hmm::HMM_MODE_FULL; sp.world = 1;
    cudaError_t e = hmm::launch_stream(D, 2, (unsigned)SP.G, sp, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? HMM_SUCCESS : HMM_ERR_CUDA;
}

// Symbol inputs: log_lik_t(d) = log_B[d][y_t] gathered on chip; lane-streaming
// kernel (OP 3 smoother, OP 4 Viterbi), D <= 8, one sequence.
hmm_status_t run_symbols(int op, int D, int V, int64_t T, const float* log_pi, const float* log_A, const float* log_B,
                         const uint8_t* y, float* filtered, float* smoothed, int32_t* path, double* scalar,
                         int32_t* info, void* ws, size_t ws_bytes, void* stream) {
    if (D < 1 || T < 1 || V < 1 || V > hmm::kStreamMaxV) return HMM_ERR_INVALID_VALUE;
    if (D > 8) return HMM_ERR_UNSUPPORTED;
    if (!log_pi || !log_A || !log_B || !y || !scalar || !info) return HMM_ERR_INVALID_VALUE;
    if (op == 0 && !smoothed) return HMM_ERR_INVALID_VALUE;
    if (op == 1 && !path) return HMM_ERR_INVALID_VALUE;
    if (!al4(log_pi) || !al4(log_A) || !al4(log_B) || !al4(y) || !al8(scalar) || !al4(info)) return HMM_ERR_INVALID_VALUE;
    if ((filtered && !al16(filtered)) || (smoothed && !al16(smoothed)) || (path && !al16(path)))
        return HMM_ERR_INVALID_VALUE;
    StPlan SP;
    if (!make_stream_plan(D, op, T, SP)) return HMM_ERR_UNSUPPORTED;
    if (!ws || ws_bytes < SP.ws_total || (reinterpret_cast<uintptr_t>(ws) & 255u)) return HMM_ERR_WORKSPACE;
    hmm::SParams sp;
    std::memset(&sp, 0, sizeof(sp));
    sp.T = T; sp.n = SP.n; sp.K = SP.K;
    sp.log_pi = log_pi; sp.log_A = log_A; sp.log_lik = nullptr;
    sp.y = y; sp.log_B = log_B; sp.V = V;
    sp.filtered = filtered; sp.smoothed = smoothed; sp.path = path; sp.scalar_out = scalar; sp.info = info;
    sp.ws = static_cast<uint8_t*>(ws);
    sp.ws_sync = SP.ws_sync; sp.ws_slots = SP.ws_slots; sp.slot_bytes = SP.slot_bytes; sp.ws_q = SP.ws_q;
    sp.ws_lagg = SP.ws_lagg; sp.ws_bp = SP.ws_bp; sp.ws_lmap = SP.ws_lmap;
    sp.L = hmm::stream_smem_layout(D, SP.G);
    sp.timers = t_timers;
    sp.mode = hmm::HMM_MODE_FULL; sp.world = 1;
    cudaError_t e = hmm::launch_stream(D, op == 0 ? 3 : 4, (unsigned)SP.G, sp, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? HMM_SUCCESS : HMM_ERR_CUDA;
}

// Split-phase scalar plumbing (hmm_dist_pack / hmm_dist_combine): one thread each.  A NULL input of
// pack contributes zeros; a NULL output of combine is not written.
__global__ void dist_pack_kernel(const uint64_t* rec, const double* lz, const double* lp, const int32_t* a,
                                 const int32_t* b, const int32_t* c, const int32_t* d, double* out) {
    out[0] = rec ? __longlong_as_double((long long)rec[0]) : 0.0;
    out[1] = rec ? __longlong_as_double((long long)rec[1]) : 0.0;
    out[2] = lz ? lz[0] : 0.0;
    out[3] = lp ? lp[0] : 0.0;
    out[4] = a ? (double)a[0] : 0.0;
    out[5] = b ? (double)b[0] : 0.0;
    out[6] = c ? (double)c[0] : 0.0;
    out[7] = d ? (double)d[0] : 0.0;
}
__device__ int32_t combine_codes(const double* g, int world, int c0) {
    bool bad = false;
    int32_t first = INT32_MAX;
    for (int r = 0; r < world; r++)
        for (int c = c0; c < c0 + 2; c++) {
            const int32_t v = (int32_t)g[(size_t)r * 8 + c];
            if (v == -1) bad = true;
            else if (v > 0 && v < first) first = v;
        }
    return bad ? -1 : (first == INT32_MAX ? 0 : first);
}
__global__ void dist_combine_kernel(int world, const double* g, uint64_t* rec_all, double* lz, double* lp,
                                    int32_t* info, int32_t* vinfo) {
    double z = 0.0, q = 0.0;
    for (int r = 0; r < world; r++) {  // rank order
        if (rec_all) {
            rec_all[2 * r] = (uint64_t)__double_as_longlong(g[(size_t)r * 8]);
            rec_all[2 * r + 1] = (uint64_t)__double_as_longlong(g[(size_t)r * 8 + 1]);
        }
        z += g[(size_t)r * 8 + 2];
        q += g[(size_t)r * 8 + 3];
    }
    if (lz) lz[0] = z;
    if (lp) lp[0] = q;
    if (info) info[0] = combine_codes(g, world, 4);
    if (vinfo) vinfo[0] = combine_codes(g, world, 6);
}

// Variable-length batches and per-sequence models.  D <= 8: the resident/chunked
// kernel with one CTA per sequence (each CTA reads its length from the offsets); D >= 9: the large-D
// engine planned for max_T (blocks and leaves past a sequence's end are empty = identity elements).
bool varlen_large_plan(int D, int op, int64_t maxT, int64_t B, LgPlan& G) {
    return make_large_plan(D, op, maxT, B, G, /*allow_tc=*/false);
}
hmm_status_t run_varlen(int op, int D, int64_t B, int64_t maxT, const int64_t* offsets, const float* log_pi,
                        const float* log_A, int per_seq, const float* log_lik, float* filtered, float* smoothed,
                        int32_t* path, double* scalar, int32_t* info, void* ws, size_t ws_bytes, void* stream) {
    if (D < 1 || B < 1 || B > 65535 || maxT < 1 || !offsets) return HMM_ERR_INVALID_VALUE;
    if (D > HMM_MAX_D) return HMM_ERR_UNSUPPORTED;
    if (!log_pi || !log_A || !log_lik || !scalar || !info) return HMM_ERR_INVALID_VALUE;
    if (op == 0 && (!smoothed || (D > 8 && !filtered))) return HMM_ERR_INVALID_VALUE;
    if (op == 1 && !path) return HMM_ERR_INVALID_VALUE;
    if (!al8(offsets) || !al4(log_pi) || !al4(log_A) || !al4(log_lik) || !al8(scalar) || !al4(info) ||
        (filtered && !al4(filtered)) || (smoothed && !al4(smoothed)) || (path && !al4(path)))
        return HMM_ERR_INVALID_VALUE;
    const int64_t pis = per_seq ? D : 0, As = per_seq ? (int64_t)D * D : 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (D > 8) {
        if (use_batchseq(D, op, B))
            return run_batchseq(op, D, maxT, B, offsets, pis, As, log_pi, log_A, log_lik, filtered, smoothed, path,
                                scalar, info, ws, ws_bytes, stream);
        LgPlan G;
        if (!varlen_large_plan(D, op, maxT, B, G)) return HMM_ERR_UNSUPPORTED;
        if (!ws || ws_bytes < G.total || (reinterpret_cast<uintptr_t>(ws) & 255u)) return HMM_ERR_WORKSPACE;
        uint8_t* w = static_cast<uint8_t*>(ws);
        hmm::LgParams lp;
        std::memset(&lp, 0, sizeof(lp));
        lp.T = maxT; lp.B = B; lp.D = D; lp.SL = G.SL; lp.NL = G.NL; lp.NB = G.NB;
        lp.log_pi = log_pi; lp.log_A = log_A; lp.log_lik = log_lik;
        lp.filtered = filtered; lp.smoothed = smoothed; lp.path = path; lp.scalar_out = scalar; lp.info = info;
        lp.ws_sync = w + G.o_sync;
        lp.leafagg = reinterpret_cast<float*>(w + G.o_leaf);
        lp.groot = reinterpret_cast<float*>(w + G.o_groot);
        lp.bpre = reinterpret_cast<float*>(w + G.o_bpre);
        lp.bsuf = reinterpret_cast<float*>(w + G.o_bsuf);
        lp.partial = reinterpret_cast<double*>(w + G.o_part);
        lp.bp = w + G.o_bp;
        lp.lmap = w + G.o_lmap;
        lp.bmap = w + G.o_bmap;
        lp.bend = reinterpret_cast<int32_t*>(w + G.o_bend);
        lp.xstar = reinterpret_cast<int32_t*>(w + G.o_xstar);
        lp.KG = G.KG; lp.NG = G.NG;
        lp.gprod = reinterpret_cast<float*>(w + G.o_gprod);
        lp.gpre = reinterpret_cast<float*>(w + G.o_gpre);
        lp.gsuf = reinterpret_cast<float*>(w + G.o_gsuf);
        lp.tc = 0;
        lp.offsets = offsets; lp.pi_stride = pis; lp.A_stride = As;
        cudaError_t e = hmm::launch_large(G.DP, op, lp, s);
        return e == cudaSuccess ? HMM_SUCCESS : HMM_ERR_CUDA;
    }
    Plan P;
    if (!make_plan(D, op, maxT, B, P, false, /*one_cta=*/true)) return HMM_ERR_UNSUPPORTED;
    if (!ws || ws_bytes < P.ws_total || (reinterpret_cast<uintptr_t>(ws) & 255u)) return HMM_ERR_WORKSPACE;
    hmm::KParams kp;
    std::memset(&kp, 0, sizeof(kp));
    kp.T = maxT; kp.R = P.R; kp.S = P.S; kp.chunk = P.chunk; kp.K = P.K; kp.KP = P.KP; kp.fused = P.fused ? 1 : 0;
    kp.log_pi = log_pi; kp.log_A = log_A; kp.log_lik = log_lik;
    kp.filtered = filtered; kp.smoothed = smoothed; kp.path = path; kp.scalar_out = scalar; kp.info = info;
    kp.ws = static_cast<uint8_t*>(ws);
    kp.ws_sync = P.ws_sync; kp.ws_slots = P.ws_slots; kp.slot_bytes = P.slot_bytes;
    kp.ws_chunk = P.ws_chunk; kp.chunk_slot = P.chunk_slot; kp.ws_bp = P.ws_bp; kp.ws_lmap = P.ws_lmap;
    kp.L = hmm::small_smem_layout(D, op, P.chunk, P.KP, P.G);
    kp.ws_cmap = P.ws_cmap;
    kp.mode = hmm::HMM_MODE_FULL; kp.world = 1;
    kp.offsets = offsets; kp.pi_stride = pis; kp.A_stride = As;
    cudaError_t e = hmm::launch_small(D, op, (unsigned)P.G, (unsigned)P.B, P.smem, false, kp, s);
    return e == cudaSuccess ? HMM_SUCCESS : HMM_ERR_CUDA;
}

size_t varlen_workspace_size(int op, int D, int64_t maxT, int64_t B) {
    if (D < 1 || D > HMM_MAX_D || maxT < 1 || B < 1 || B > 65535) return 0;
    if (D > 8) {
        LgPlan G;
        if (!varlen_large_plan(D, op, maxT, B, G)) return 0;
        size_t w = G.total;
        if (bs_dp(D) && bs_workspace(op, D, maxT, B) > w) w = bs_workspace(op, D, maxT, B);
        return w;
    }
    Plan P;
    return make_plan(D, op, maxT, B, P, false, true) ? P.ws_total : 0;
}

}  // namespace

extern "C" {

hmm_status_t hmm_dist_pack(const void* record16, const double* log_z_partial, const double* log_prob_partial,
                           const int32_t* s_info_reduce, const int32_t* s_info_finish, const int32_t* v_info_reduce,
                           const int32_t* v_info_forward, double* packed8, void* stream) {
    if (!packed8 || !al8(packed8) || (record16 && !al8(record16)) || (log_z_partial && !al8(log_z_partial)) ||
        (log_prob_partial && !al8(log_prob_partial)) || (s_info_reduce && !al4(s_info_reduce)) ||
        (s_info_finish && !al4(s_info_finish)) || (v_info_reduce && !al4(v_info_reduce)) ||
        (v_info_forward && !al4(v_info_forward)))
        return HMM_ERR_INVALID_VALUE;
    dist_pack_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint64_t*>(record16), log_z_partial, log_prob_partial, s_info_reduce, s_info_finish,
        v_info_reduce, v_info_forward, packed8);
    return cudaGetLastError() == cudaSuccess ? HMM_SUCCESS : HMM_ERR_CUDA;
}

hmm_status_t hmm_dist_combine(int world, const double* gathered, void* records_all, double* log_z,
                              double* log_prob, int32_t* info, int32_t* vinfo, void* stream) {
    if (world < 1 || !gathered || !al8(gathered) || (records_all && !al8(records_all)) || (log_z && !al8(log_z)) ||
        (log_prob && !al8(log_prob)) || (info && !al4(info)) || (vinfo && !al4(vinfo)))
        return HMM_ERR_INVALID_VALUE;
    dist_combine_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(
        world, gathered, static_cast<uint64_t*>(records_all), log_z, log_prob, info, vinfo);
    return cudaGetLastError() == cudaSuccess ? HMM_SUCCESS : HMM_ERR_CUDA;
}

const char* hmm_status_string(hmm_status_t status) {
    switch (status) {
        case HMM_SUCCESS: return "HMM_SUCCESS";
        case HMM_ERR_INVALID_VALUE: return "HMM_ERR_INVALID_VALUE";
        case HMM_ERR_WORKSPACE: return "HMM_ERR_WORKSPACE";
        case HMM_ERR_UNSUPPORTED: return "HMM_ERR_UNSUPPORTED";
        case HMM_ERR_CUDA: return "HMM_ERR_CUDA";
        default: return "HMM_ERR_UNKNOWN";
    }
}

const char* hmm_version(void) { return "hmmscan 0.1 sm_100a"; }

void hmm_debug_set_timers(unsigned long long* device_buf) { t_timers = device_buf; }

void hmm_debug_force_path(int path) { t_force_path = (path >= 0 && path <= 6) ? path : 0; }

int hmm_debug_plan(int op, int D, int64_t T, int64_t B, int64_t* out /*[8]*/) {
    StPlan SP;
    if (use_stream(D, T, B, false) && make_stream_plan(D, op, T, SP)) {
        out[0] = SP.G; out[1] = SP.n; out[2] = hmm::stream_s(D); out[3] = hmm::stream_s(D); out[4] = SP.K;
        out[5] = 2; out[6] = (int64_t)SP.smem; out[7] = hmm::stream_nt(D);
        return 1;
    }
    Plan P;
    if (!make_plan(D, op, T, B, P)) return 0;
    out[0] = P.G; out[1] = P.R; out[2] = P.S; out[3] = P.chunk; out[4] = P.K; out[5] = P.fused;
    out[6] = (int64_t)P.smem; out[7] = P.NT;
    return 1;
}

size_t hmm_workspace_size(int op, int D, int64_t T, int64_t B) {
    if (op == HMM_OP_VITERBI_MAXPRODUCT || op == HMM_OP_VITERBI_PATHELEM)
        return hmm::variants_workspace_size(op, D, T, B);
    if (op == HMM_OP_SMOOTH_VARLEN || op == HMM_OP_VITERBI_VARLEN)
        return varlen_workspace_size(op == HMM_OP_SMOOTH_VARLEN ? 0 : 1, D, T, B);
    if (op == 2) {  // smoother with E-step statistics (hmm_smooth_stats)
        StPlan SP;
        if (D < 1 || D > 8 || T < 1 || B != 1 || !make_stream_plan(D, 2, T, SP)) return 0;
        return SP.ws_total;
    }
    if ((op != 0 && op != 1) || D < 1 || D > HMM_MAX_D || T < 1 || B < 1) return 0;
    if (D > 8) {  // any large-D engine may run (hmm_debug_force_path): size for all of them
        LgPlan G, H2;
        if (!make_large_plan(D, op, T, B, G, true) || !make_large_plan(D, op, T, B, H2, false)) return 0;
        size_t w = G.total > H2.total ? G.total : H2.total;
        if (bs_dp(D) && bs_workspace(op, D, T, B) > w) w = bs_workspace(op, D, T, B);
        return w;
    }
    Plan P;
    if (!make_plan(D, op, T, B, P)) return 0;
    size_t w = P.ws_total;
    StPlan SP;
    if (B == 1 && D <= 8 && make_stream_plan(D, op, T, SP) && SP.ws_total > w) w = SP.ws_total;
    return w;
}

hmm_status_t hmm_smooth(int D, int64_t T, const float* log_pi, const float* log_A, const float* log_lik,
                        float* filtered, float* smoothed, double* log_likelihood, int32_t* info, void* workspace,
                        size_t workspace_bytes, void* stream) {
    return run(0, D, T, 1, log_pi, log_A, log_lik, filtered, smoothed, nullptr, log_likelihood, info, workspace,
               workspace_bytes, stream);
}

hmm_status_t hmm_smooth_stats(int D, int64_t T, const float* log_pi, const float* log_A, const float* log_lik,
                              float* filtered, float* smoothed, double* log_likelihood, double* xi_sum,
                              double* gamma_sum, int32_t* info, void* workspace, size_t workspace_bytes, void* stream) {
    return run_stats(D, T, log_pi, log_A, log_lik, filtered, smoothed, log_likelihood, xi_sum, gamma_sum, info,
                     workspace, workspace_bytes, stream);
}

hmm_status_t hmm_smooth_symbols(int D, int V, int64_t T, const float* log_pi, const float* log_A, const float* log_B,
                                const uint8_t* y, float* filtered, float* smoothed, double* log_likelihood, int32_t* info,
                                void* workspace, size_t workspace_bytes, void* stream) {
    return run_symbols(0, D, V, T, log_pi, log_A, log_B, y, filtered, smoothed, nullptr, log_likelihood, info,
                       workspace, workspace_bytes, stream);
}

hmm_status_t hmm_viterbi_symbols(int D, int V, int64_t T, const float* log_pi, const float* log_A, const float* log_B,
                                 const uint8_t* y, int32_t* path, double* log_prob, int32_t* info, void* workspace,
                                 size_t workspace_bytes, void* stream) {
    return run_symbols(1, D, V, T, log_pi, log_A, log_B, y, nullptr, nullptr, path, log_prob, info, workspace,
                       workspace_bytes, stream);
}

hmm_status_t hmm_viterbi(int D, int64_t T, const float* log_pi, const float* log_A, const float* log_lik,
                         int32_t* path, double* log_prob, int32_t* info, void* workspace, size_t workspace_bytes,
                         void* stream) {
    return run(1, D, T, 1, log_pi, log_A, log_lik, nullptr, nullptr, path, log_prob, info, workspace,
               workspace_bytes, stream);
}

size_t hmm_dist_agg_bytes(int D) {
    if (D < 1 || D > HMM_MAX_D) return 0;
    if (D <= 8) return hmm::align16((size_t)D * D * 4);
    const size_t DP = D <= 16 ? 16 : (D <= 32 ? 32 : 64);  // large-D aggregates: padded DP x DP floats
    return DP * DP * 4;
}

size_t hmm_dist_record_bytes(void) { return 16; }

size_t hmm_dist_record_bytes_d(int D) {
    if (D < 1 || D > HMM_MAX_D) return 0;
    if (D <= 8) return 16;
    const size_t DP = D <= 16 ? 16 : (D <= 32 ? 32 : 64);
    return DP + 16;  // uint8 map[DP], int32 x* at byte DP, padded to 16
}

size_t hmm_dist_workspace_size(int op, int D, int64_t T_local) {
    if ((op != 0 && op != 1) || D < 1 || D > HMM_MAX_D || T_local < 1) return 0;
    if (D > 8) {  // split phase at D > 8: the large-D block scan
        LgPlan G;
        return make_large_plan(D, op, T_local, 1, G) ? G.total : 0;
    }
    Plan P;
    if (!make_plan(D, op, T_local, 1, P, true)) return 0;
    size_t w = P.ws_total;
    StPlan SP;
    if (make_stream_plan(D, op, T_local, SP) && SP.ws_total > w) w = SP.ws_total;
    return w;
}

hmm_status_t hmm_smooth_dist_reduce(int D, int64_t T_local, int64_t t_base, const float* log_pi, const float* log_A,
                                    const float* log_lik, void* agg_out, int32_t* info, void* workspace,
                                    size_t workspace_bytes, void* stream) {
    if (!agg_out || (reinterpret_cast<uintptr_t>(agg_out) & 15u)) return HMM_ERR_INVALID_VALUE;
    DistArgs da; da.mode = hmm::HMM_MODE_REDUCE; da.t_base = t_base; da.agg_out = static_cast<float*>(agg_out);
    return run(0, D, T_local, 1, log_pi, log_A, log_lik, nullptr, nullptr, nullptr, nullptr, info, workspace,
               workspace_bytes, stream, da);
}

hmm_status_t hmm_smooth_dist_finish(int D, int64_t T_local, int64_t t_base, const float* log_pi, const float* log_A,
                                    const float* log_lik, const void* agg_all, int rank, int world, float* filtered,
                                    float* smoothed, double* log_z_partial, int32_t* info, void* workspace,
                                    size_t workspace_bytes, void* stream) {
    if (!agg_all) return HMM_ERR_INVALID_VALUE;
    DistArgs da; da.mode = hmm::HMM_MODE_SFINISH; da.t_base = t_base; da.rank = rank; da.world = world;
    da.agg_all = static_cast<const float*>(agg_all);
    return run(0, D, T_local, 1, log_pi, log_A, log_lik, filtered, smoothed, nullptr, log_z_partial, info, workspace,
               workspace_bytes, stream, da);
}

hmm_status_t hmm_viterbi_dist_reduce(int D, int64_t T_local, int64_t t_base, const float* log_pi, const float* log_A,
                                     const float* log_lik, void* agg_out, int32_t* info, void* workspace,
                                     size_t workspace_bytes, void* stream) {
    if (!agg_out || (reinterpret_cast<uintptr_t>(agg_out) & 15u)) return HMM_ERR_INVALID_VALUE;
    DistArgs da; da.mode = hmm::HMM_MODE_REDUCE; da.t_base = t_base; da.agg_out = static_cast<float*>(agg_out);
    return run(1, D, T_local, 1, log_pi, log_A, log_lik, nullptr, nullptr, nullptr, nullptr, info, workspace,
               workspace_bytes, stream, da);
}

hmm_status_t hmm_viterbi_dist_forward(int D, int64_t T_local, int64_t t_base, const float* log_pi,
                                      const float* log_A, const float* log_lik, const void* agg_all, int rank,
                                      int world, void* record_out, double* log_prob_partial, int32_t* info,
                                      void* workspace, size_t workspace_bytes, void* stream) {
    if (!agg_all || !record_out || (reinterpret_cast<uintptr_t>(record_out) & 15u)) return HMM_ERR_INVALID_VALUE;
    DistArgs da; da.mode = hmm::HMM_MODE_VFORWARD; da.t_base = t_base; da.rank = rank; da.world = world;
    da.agg_all = static_cast<const float*>(agg_all); da.rec_out = static_cast<uint8_t*>(record_out);
    return run(1, D, T_local, 1, log_pi, log_A, log_lik, nullptr, nullptr, nullptr, log_prob_partial, info,
               workspace, workspace_bytes, stream, da);
}

hmm_status_t hmm_viterbi_dist_finish(int D, int64_t T_local, int64_t t_base, const float* log_pi, const float* log_A,
                                     const float* log_lik, const void* records_all, int rank, int world,
                                     int32_t* path, int32_t* info, void* workspace, size_t workspace_bytes,
                                     void* stream) {
    if (!records_all) return HMM_ERR_INVALID_VALUE;
    DistArgs da; da.mode = hmm::HMM_MODE_VFINISH; da.t_base = t_base; da.rank = rank; da.world = world;
    da.rec_all = static_cast<const uint8_t*>(records_all);
    return run(1, D, T_local, 1, log_pi, log_A, log_lik, nullptr, nullptr, path, nullptr, info, workspace,
               workspace_bytes, stream, da);
}

hmm_status_t hmm_smooth_batched(int D, int64_t T, int64_t B, const float* log_pi, const float* log_A,
                                const float* log_lik, float* filtered, float* smoothed, double* log_likelihood,
                                int32_t* info, void* workspace, size_t workspace_bytes, void* stream) {
    return run(0, D, T, B, log_pi, log_A, log_lik, filtered, smoothed, nullptr, log_likelihood, info, workspace,
               workspace_bytes, stream);
}

hmm_status_t hmm_viterbi_batched(int D, int64_t T, int64_t B, const float* log_pi, const float* log_A,
                                 const float* log_lik, int32_t* path, double* log_prob, int32_t* info,
                                 void* workspace, size_t workspace_bytes, void* stream) {
    return run(1, D, T, B, log_pi, log_A, log_lik, nullptr, nullptr, path, log_prob, info, workspace,
               workspace_bytes, stream);
}

}  // extern "C"

hmm_status_t hmm_smooth_varlen(int D, int64_t B, int64_t max_T, const int64_t* offsets, const float* log_pi,
                               const float* log_A, int per_sequence_model, const float* log_lik, float* filtered,
                               float* smoothed, double* log_likelihood, int32_t* info, void* workspace,
                               size_t workspace_bytes, void* stream) {
    return run_varlen(0, D, B, max_T, offsets, log_pi, log_A, per_sequence_model, log_lik, filtered, smoothed,
                      nullptr, log_likelihood, info, workspace, workspace_bytes, stream);
}

hmm_status_t hmm_viterbi_varlen(int D, int64_t B, int64_t max_T, const int64_t* offsets, const float* log_pi,
                                const float* log_A, int per_sequence_model, const float* log_lik, int32_t* path,
                                double* log_prob, int32_t* info, void* workspace, size_t workspace_bytes,
                                void* stream) {
    return run_varlen(1, D, B, max_T, offsets, log_pi, log_A, per_sequence_model, log_lik, nullptr, nullptr, path,
                      log_prob, info, workspace, workspace_bytes, stream);
}
