// hmm_large.h — parameter block of the large-D kernels (hmm_large.cu), filled by hmm_abi.cu.
#pragma once
#include <cstddef>
#include <cstdint>

namespace hmm {

struct LgParams {
    int64_t T, B;
    int D;
    int64_t SL;  // steps per leaf
    int64_t NL;  // leaves per sequence
    int64_t NB;  // blocks (CTAs of K1/K3) per sequence
    const float* log_pi;
    const float* log_A;
    const float* log_lik;
    float* filtered;
    float* smoothed;
    int32_t* path;
    double* scalar_out;
    int32_t* info;
    // workspace views
    uint8_t* ws_sync;   // [B][64 B]
    float* leafagg;     // [B][NL][DP*DP]
    float* groot;       // [B][NB][DP*DP]
    float* bpre;        // [B][NB][DP]
    float* bsuf;        // [B][NB][DP]
    double* partial;    // [B][NL]
    uint8_t* bp;        // [B][T][DP]   Viterbi backpointers
    uint8_t* lmap;      // [B][NL][DP]  Viterbi leaf maps
    uint8_t* bmap;      // [B][NB][DP]  Viterbi block maps
    int32_t* bend;      // [B][NB]      Viterbi block end states
    int32_t* xstar;     // [B]
    // tensor-core leaf products (sum-product, DP = 64): hmm_large_tc.cu
    int tc;             // 1: leaf aggregates come from lg_leaf_tc_kernel
    float* lik;         // [B][T][64] likelihood rows exp(ll - m_t), padded with 0
    // variable-length batches / per-sequence models (see KParams in hmm_plan.h)
    const int64_t* offsets;
    int64_t pi_stride, A_stride;
    // two-level carry (NG > 1): KG block roots per group, group products and their carries
    int64_t KG, NG;
    float* gprod;  // [B][NG][DP*DP]
    float* gpre;   // [B][NG][DP]
    float* gsuf;   // [B][NG][DP]
    // split-phase distributed smoother (B = 1; hmm_plan.h HMM_MODE_*): this rank's global offset, the
    // gathered rank aggregates (DP x DP floats each), the rank aggregate out, the rank carries [2][DP]
    int mode;
    int64_t t_base;
    int rank, world;
    const float* agg_all;
    float* agg_out;
    float* rcar;
    uint8_t* rec_out;       // Viterbi forward: this rank's record {uint8 map[DP], int32 x* at byte DP}
    const uint8_t* rec_all; // Viterbi finish: the gathered records, rec_bytes apart
    int rec_bytes;
};

// Batch-parallel plan (hmm_batchseq.cu): one lane group per sequence, 9 <= D <= 32.
struct BSParams {
    int64_t T, B;
    int D;
    const float* log_pi;
    const float* log_A;
    const float* log_lik;
    float* filtered;
    float* smoothed;
    int32_t* path;
    double* scalar_out;
    int32_t* info;
    uint8_t* bp;  // [B][T][DP] Viterbi backpointers (workspace)
    float* sbeta;       // bidirectional smoother: [B][s_rows][D] backward potentials of each second half
    int64_t s_rows;
    const int64_t* offsets;
    int64_t pi_stride, A_stride;
};

}  // namespace hmm
