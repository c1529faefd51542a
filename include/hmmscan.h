/*
 * hmmscan.h — C ABI of the B200-native temporally parallel HMM inference library (libhmmscan.so).
 *
 * Implements the parallel sum-product smoother (Algorithm 3) and the parallel
 * max-product MAP estimator (Definition 5 + Propositions 2-3, with argmax
 * backpointers instead of Eq. 21's per-step assembly, see DESIGN.md "Readings" #6) for the HMM of
 * Eqs. 4-6, on sm_100a.  All compute runs in this library's CUDA kernels.
 *
 * Conventions (all functions):
 *   - D      number of states, 1 <= D <= HMM_MAX_D.
 *   - T      number of time steps (>= 1); t is 0-based here (the paper is 1-based).
 *   - log_pi [D]      fp32, log p(x_0 = d)                                  (prior)
 *   - log_A  [D*D]    fp32 row-major, log_A[i*D+j] = log p(x_t=j | x_{t-1}=i)
 *   - log_lik[T*D]    fp32 row-major, log p(y_t | x_t = d)
 *     Inputs are general log-potentials: they need not be normalised; -inf is allowed anywhere
 *     (a forbidden transition / impossible observation).  NaN and +inf are errors (info = -1).
 *   - The potentials are psi_0(x_0) = exp(log_pi + log_lik_0) and
 *     psi_t(x_{t-1}, x_t) = exp(log_A + log_lik_t) (Eq. 5).
 *   - ALL data pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors) unless the function
 *     name says _host.  Scalars outputs (log_likelihood, log_prob, info) are device words too.
 *   - Every call is asynchronous and stream-ordered on `stream` (a cudaStream_t; NULL = legacy
 *     default stream).  Nothing is allocated or freed by the library and no host sync happens.
 *   - workspace: caller-owned device memory of at least hmm_workspace_size(...) bytes, ZERO-FILLED
 *     ONCE when allocated.  The kernels leave it in its zero state again when they finish, so the
 *     same workspace can be reused by later calls on the same stream without re-zeroing.  Two calls
 *     that may run concurrently (different streams) need different workspaces.
 *   - Determinism: fixed reduction trees; the same inputs, sizes and device give bitwise-identical
 *     outputs run to run.
 *
 * Errors:
 *   - Host-detected, synchronous, returned: HMM_ERR_INVALID_VALUE (bad sizes, NULL pointer, pointer
 *     not 4-byte aligned), HMM_ERR_WORKSPACE (workspace too small or NULL), HMM_ERR_UNSUPPORTED
 *     (shape not supported by this build, e.g. T beyond the per-CTA chunk limit), HMM_ERR_CUDA (a
 *     launch failed; cudaGetLastError() has the detail).
 *   - Device-detected, asynchronous, written to info[b]: 0 = ok; t+1 = the smallest t at which no
 *     state sequence is consistent with the evidence and the transitions up to t (zero forward mass
 *     for the smoother, all V_t = -inf for Viterbi); -1 = a NaN or +inf input.
 *     When info != 0 the other outputs of that sequence are undefined (cuSOLVER devInfo idiom).
 *   - Kernels whose CTAs meet at a grid barrier bound the wait (4 s): a barrier that can never
 *     complete (a workspace left dirty by an aborted or faulted launch, or a CTA that is not resident)
 *     traps instead of hanging the device.  The stream then reports cudaErrorLaunchFailure, the CUDA
 *     context is unusable, and any workspace used by a failed call must be zero-filled again before
 *     reuse (the kernels only restore the zero state on successful completion).
 *   - Threading: any host thread may call; the per-device kernel-attribute record is mutex-guarded, so
 *     concurrent first calls and several GPUs in one process are safe (one workspace per concurrent
 *     call).
 */
#ifndef HMMSCAN_H
#define HMMSCAN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HMM_MAX_D 64

typedef enum {
    HMM_SUCCESS = 0,
    HMM_ERR_INVALID_VALUE = 1,
    HMM_ERR_WORKSPACE = 2,
    HMM_ERR_UNSUPPORTED = 3,
    HMM_ERR_CUDA = 4
} hmm_status_t;

typedef enum {
    HMM_OP_SMOOTH = 0,
    HMM_OP_VITERBI = 1,
    HMM_OP_SMOOTH_STATS = 2,
    HMM_OP_VITERBI_MAXPRODUCT = 5, /* hmm_viterbi_maxproduct (Algorithm 5) */
    HMM_OP_VITERBI_PATHELEM = 6,   /* hmm_viterbi_path_elements (Definition 4) */
    HMM_OP_SMOOTH_VARLEN = 7,      /* hmm_smooth_varlen (T = max_T) */
    HMM_OP_VITERBI_VARLEN = 8      /* hmm_viterbi_varlen (T = max_T) */
} hmm_op_t;

/* Device info codes beyond the common ones (0 ok, t+1 first impossible step, -1 NaN / +inf input). */
#define HMM_INFO_AMBIGUOUS (-2) /* Algorithm 5: the Eq. 21 assembly is not a MAP path (ties) */
#define HMM_INFO_NO_PATH (-3)   /* Definition 4: no sequence has nonzero weight (step not located) */
#define HMM_INFO_BAD_LENGTH (-4) /* varlen batches: offsets[b+1] - offsets[b] outside [1, max_T] */
#define HMM_PATHELEM_MAX_T 1024 /* cap of the path-element reduction */

/* Human-readable name of a status code (static storage, never NULL). */
const char* hmm_status_string(hmm_status_t status);

/* Library version string, e.g. "hmmscan 0.1 sm_100a". */
const char* hmm_version(void);

/* Bytes of device workspace needed by the hmm_smooth and hmm_viterbi families for (op, D, T, B) on the current
 * device (op = HMM_OP_SMOOTH_STATS: hmm_smooth_stats, B = 1).  Returns 0 for invalid arguments.  The value
 * depends on the device's SM count. */
size_t hmm_workspace_size(int op, int D, int64_t T, int64_t B);

/*
 * Parallel sum-product smoother — Algorithm 3.
 *   filtered [T*D] out: p(x_t | y_0..y_t), the normalised forward potential a_{0:t} (Thm 1,
 *                       PAPER.md:304-341; filtering PAPER.md:177).  May be NULL (not written) for
 *                       D <= 8; required for D > 8 (the large-D path stages alpha there).
 *   smoothed [T*D] out: p(x_t | y_0..y_{T-1}) = a_{0:t} a_{t:T+1} / Z_t (Eq. 14).
 *   log_likelihood [1] out (double): log Z, Z the partition function of Eq. 1
 *                       = log p(y_0..y_{T-1}) when the inputs are normalised probabilities.
 *   info [1] out (int32): see Errors.
 */
hmm_status_t hmm_smooth(int D, int64_t T, const float* log_pi, const float* log_A, const float* log_lik,
                        float* filtered, float* smoothed, double* log_likelihood, int32_t* info,
                        void* workspace, size_t workspace_bytes, void* stream);

/*
 * Smoother + Baum-Welch expectation statistics ("in expectation step, BWA uses the
 * forward-backward algorithm, which can be parallelized using the methods proposed in this article").
 * Same outputs as hmm_smooth (filtered and smoothed may both be NULL: statistics only) plus
 *   xi_sum [D*D] out (double): sum_{t=1..T-1} p(x_{t-1}=i, x_t=j | y), the pairwise posteriors of the
 *                       factorisation Eq. 6 from the forward / backward potentials
 *                       (row-major, i = previous state);
 *   gamma_sum [D] out (double): sum_{t=0..T-1} p(x_t=d | y) (Eq. 14).
 * The M-step transition update is A'(i,j) = xi_sum(i,j) / sum_j xi_sum(i,j).  1 <= D <= 8, one
 * sequence; log_lik / filtered / smoothed must be 16-byte aligned (HMM_ERR_INVALID_VALUE otherwise),
 * D > 8 -> HMM_ERR_UNSUPPORTED.  Workspace: hmm_workspace_size(HMM_OP_SMOOTH_STATS, D, T, 1).
 * Statistics are fp32 per 16-step slice, fp64 across slices, summed in a fixed order (deterministic).
 */
hmm_status_t hmm_smooth_stats(int D, int64_t T, const float* log_pi, const float* log_A, const float* log_lik,
                              float* filtered, float* smoothed, double* log_likelihood, double* xi_sum,
                              double* gamma_sum, int32_t* info, void* workspace, size_t workspace_bytes,
                              void* stream);

/*
 * Symbol-input variants: discrete observations y_t in [0, V) with emission matrix
 * log_B[d*V + v] = log p(y_t = v | x_t = d) (the O matrix of the paper's GE channel);
 * the elements use log_lik_t(d) = log_B[d*V + y_t] (Eq. 5b), gathered on chip from a table, so the
 * input is 1 byte per step instead of 4*D.  Outputs and semantics as hmm_smooth / hmm_viterbi.
 * 1 <= D <= 8, 1 <= V <= 256, one sequence; y 4-byte aligned, outputs 16-byte aligned.  A symbol
 * >= V or a NaN / +inf entry of log_B is reported as info = -1.  Workspace:
 * hmm_workspace_size(HMM_OP_SMOOTH or HMM_OP_VITERBI, D, T, 1).
 */
hmm_status_t hmm_smooth_symbols(int D, int V, int64_t T, const float* log_pi, const float* log_A, const float* log_B,
                                const uint8_t* y, float* filtered, float* smoothed, double* log_likelihood,
                                int32_t* info, void* workspace, size_t workspace_bytes, void* stream);
hmm_status_t hmm_viterbi_symbols(int D, int V, int64_t T, const float* log_pi, const float* log_A, const float* log_B,
                                 const uint8_t* y, int32_t* path, double* log_prob, int32_t* info, void* workspace,
                                 size_t workspace_bytes, void* stream);

/*
 * Parallel max-product MAP (Viterbi) — Definition 5 / Propositions 2-3 for the
 * forward max-potentials, argmax backpointers (Alg. 4 line 5) and a parallel
 * backtrack by composition of chunk backpointer maps (DESIGN.md §"Viterbi").
 *   path [T] out (int32): argmax_x log p(x, y) (Eq. 17); ties broken towards the
 *                         smallest state index in every argmax (reading 5).
 *   log_prob [1] out (double): the joint log p(x*, y) = max of the forward max-potential at T-1
 *                         (Eqs. 16-17, Corollary 1 PAPER.md:621-632) — not the posterior.
 */
hmm_status_t hmm_viterbi(int D, int64_t T, const float* log_pi, const float* log_A, const float* log_lik,
                         int32_t* path, double* log_prob, int32_t* info,
                         void* workspace, size_t workspace_bytes, void* stream);

/*
 * Batched variants: B independent sequences of equal length T sharing log_pi and log_A.
 *   log_lik [B*T*D], filtered/smoothed [B*T*D], log_likelihood [B], path [B*T], log_prob [B], info [B].
 */
hmm_status_t hmm_smooth_batched(int D, int64_t T, int64_t B, const float* log_pi, const float* log_A,
                                const float* log_lik, float* filtered, float* smoothed,
                                double* log_likelihood, int32_t* info,
                                void* workspace, size_t workspace_bytes, void* stream);

hmm_status_t hmm_viterbi_batched(int D, int64_t T, int64_t B, const float* log_pi, const float* log_A,
                                 const float* log_lik, int32_t* path, double* log_prob, int32_t* info,
                                 void* workspace, size_t workspace_bytes, void* stream);

/*
 * Variable-length batches and per-sequence models (extends the batched calls).
 * B independent sequences packed back to back: sequence b owns rows [offsets[b], offsets[b+1]) of
 * log_lik [N*D] (N = offsets[B]) and of the outputs filtered / smoothed [N*D] and path [N]; its length
 * T_b = offsets[b+1] - offsets[b] must lie in [1, max_T] (else info[b] = HMM_INFO_BAD_LENGTH and that
 * sequence's outputs are undefined).  Every sequence is its own HMM (Eq. 5 potentials):
 * its first step takes the prior, its last step the all-ones backward element a_{T:T+1} (Thm 2).
 *   offsets [B+1] in: device int64, 8-B aligned (read on the device; the host passes only max_T).
 *   per_sequence_model = 0: log_pi [D], log_A [D*D] shared by the batch;
 *                      != 0: log_pi [B*D], log_A [B*D*D], one model per sequence.
 *   log_likelihood / log_prob / info [B] out, as the batched calls.
 * 1 <= D <= 64 (D >= 9: filtered is required, as hmm_smooth).  D <= 8 runs one CTA per sequence; D >= 9
 * the large-D block scan planned for max_T (CUDA cores; the tensor-core leaf needs one shared A).
 * Workspace: hmm_workspace_size(HMM_OP_SMOOTH_VARLEN / HMM_OP_VITERBI_VARLEN, D, max_T, B), zero-filled,
 * left zeroed.
 */
hmm_status_t hmm_smooth_varlen(int D, int64_t B, int64_t max_T, const int64_t* offsets, const float* log_pi,
                               const float* log_A, int per_sequence_model, const float* log_lik, float* filtered,
                               float* smoothed, double* log_likelihood, int32_t* info, void* workspace,
                               size_t workspace_bytes, void* stream);

hmm_status_t hmm_viterbi_varlen(int D, int64_t B, int64_t max_T, const int64_t* offsets, const float* log_pi,
                                const float* log_A, int per_sequence_model, const float* log_lik, int32_t* path,
                                double* log_prob, int32_t* info, void* workspace, size_t workspace_bytes,
                                void* stream);

/*
 * Paper-faithful Viterbi variants (validation modes, not the production path).
 * 1 <= D <= 8, B sequences of equal length T sharing log_pi / log_A (layouts as the batched calls; B = 1
 * for a single sequence).  Inputs/outputs are device pointers, 4-B aligned (doubles / int64 8-B aligned).
 *
 * hmm_viterbi_maxproduct — Algorithm 5: forward max-product scan -> log psi~f_k
 * (Prop. 2), reversed scan -> log psi~b_k (Prop. 3), then
 * x*_k = argmax_x psi~f_k(x) psi~b_k(x) (Theorem 4 / Eq. 21), smallest index on ties.
 *   path [B*T] out: the Eq. 21 assembly.  Under exact ties it need not be ONE path.
 *   log_prob [B] out (double): the per-step optimum max_x log psi~f_k + log psi~b_k (k = T-1), = the MAP
 *                         joint log-probability by Theorem 4.
 *   path_weight [B] out (double, may be NULL): Eq. 6 joint log-weight of the assembled path, fp64.
 *   n_tied [B] out (int64, may be NULL): steps whose best and second-best max-marginal scores differ by
 *                         <= tie_tol (nats, >= 0; 0 counts exact fp32 ties).
 *   info [B] out: as hmm_viterbi, plus HMM_INFO_AMBIGUOUS when path_weight < log_prob - 1e-6 max(1, |log_prob|)
 *                         (SPEC.md:297-303's coherence diagnostic: the tied steps did not assemble into a
 *                         MAP path).
 *   Workspace: hmm_workspace_size(HMM_OP_VITERBI_MAXPRODUCT, D, T, B), zero-filled, left zeroed.
 *
 * hmm_viterbi_path_elements — Definition 4: elements a~_{i:j} = (A_{i:j}, X^_{i:j})
 * carrying the max weight and the interior path for every state pair, combined by v; the reduction
 * a~_{0:T+1} holds the MAP weight and path (Theorem 3, Corollary 1).  Memory grows as
 * D^2 states per step, so T <= HMM_PATHELEM_MAX_T (else HMM_ERR_INVALID_VALUE).
 *   path [B*T] out: the MAP path (smallest x^_j at every combine on ties); log_prob [B] out (double).
 *   info [B] out: 0, -1 (NaN / +inf input) or HMM_INFO_NO_PATH (every sequence has zero weight).
 *   Workspace: hmm_workspace_size(HMM_OP_VITERBI_PATHELEM, D, T, B) (no zero-fill needed).
 */
hmm_status_t hmm_viterbi_maxproduct(int D, int64_t T, int64_t B, const float* log_pi, const float* log_A,
                                    const float* log_lik, float tie_tol, int32_t* path, double* log_prob,
                                    double* path_weight, int64_t* n_tied, int32_t* info, void* workspace,
                                    size_t workspace_bytes, void* stream);

hmm_status_t hmm_viterbi_path_elements(int D, int64_t T, int64_t B, const float* log_pi, const float* log_A,
                                       const float* log_lik, int32_t* path, double* log_prob, int32_t* info,
                                       void* workspace, size_t workspace_bytes, void* stream);

/*
 * Split-phase distributed execution (one sequence partitioned along T across `world` ranks, one
 * process per GPU).  Rank r owns the contiguous global steps
 * [t_base, t_base + T_local) and passes its slice of log_lik.  The library never calls NCCL: between
 * the phases the CALLER all-gathers small fixed-size blobs (e.g. torch.distributed
 * all_gather_into_tensor over NCCL/NVLink) into rank order.  All phases of one rank must use the same
 * workspace (hmm_dist_workspace_size bytes, zero-filled once), on the same stream, in order.
 * Supported for a single sequence, 1 <= D <= 64.  hmm_dist_agg_bytes(D) is align16(D*D*4) for D <= 8
 * and DP*DP*4 (DP = 16, 32 or 64, the padded state count) for D > 8.  The Viterbi rank record is
 * hmm_dist_record_bytes_d(D) bytes: 16 for D <= 8 (u64 byte map, i32 x*; hmm_dist_record_bytes()), and
 * DP + 16 for D > 8 (uint8 map[DP], i32 x* at byte DP); hmm_dist_pack / hmm_dist_combine carry only the
 * 16-byte records, so at D > 8 the caller all-gathers the records itself.
 *
 * Smoother (Algorithm 3 across ranks; the rank aggregate is the ordered product of the rank's
 * elements, Def. 3 / PAPER.md:281-290):
 *   1. hmm_smooth_dist_reduce  -> agg_out (hmm_dist_agg_bytes(D) bytes, 16-B aligned device memory)
 *   2. caller: all-gather the world aggregates -> agg_all[world] (rank order)
 *   3. hmm_smooth_dist_finish  -> filtered/smoothed of the local slice, log_z_partial[1] (double).
 *      log Z = sum over ranks of log_z_partial, in rank order (caller: all-gather + sum).
 * Viterbi (Def. 5 aggregates; rank backpointer maps compose right to left):
 *   1. hmm_viterbi_dist_reduce  -> agg_out
 *   2. caller: all-gather -> agg_all
 *   3. hmm_viterbi_dist_forward -> record_out (hmm_dist_record_bytes_d(D) bytes, see above),
 *      log_prob_partial[1]; log_prob = sum of partials over ranks.
 *   4. caller: all-gather the records -> records_all[world]
 *   5. hmm_viterbi_dist_finish  -> path of the local slice.
 * info: reduce reports bad inputs (-1); smoother finish / Viterbi forward report the first impossible
 * GLOBAL step + 1; hmm_viterbi_dist_finish only backtracks and always writes info = 0.
 * Kernel choice: every phase of a rank must run the same decomposition (later phases read the workspace
 * layout the reduce call wrote), so it is chosen from log_lik's alignment alone: 16-B aligned log_lik
 * selects the lane-streaming kernel, and then filtered / smoothed / path must be 16-B aligned too
 * (HMM_ERR_INVALID_VALUE otherwise); a log_lik that is only 4-B aligned selects the chunked kernel in
 * every phase.
 */
size_t hmm_dist_agg_bytes(int D);
size_t hmm_dist_record_bytes(void);
size_t hmm_dist_record_bytes_d(int D);
size_t hmm_dist_workspace_size(int op, int D, int64_t T_local);
hmm_status_t hmm_smooth_dist_reduce(int D, int64_t T_local, int64_t t_base, const float* log_pi, const float* log_A,
                                    const float* log_lik, void* agg_out, int32_t* info, void* workspace,
                                    size_t workspace_bytes, void* stream);
hmm_status_t hmm_smooth_dist_finish(int D, int64_t T_local, int64_t t_base, const float* log_pi, const float* log_A,
                                    const float* log_lik, const void* agg_all, int rank, int world, float* filtered,
                                    float* smoothed, double* log_z_partial, int32_t* info, void* workspace,
                                    size_t workspace_bytes, void* stream);
hmm_status_t hmm_viterbi_dist_reduce(int D, int64_t T_local, int64_t t_base, const float* log_pi, const float* log_A,
                                     const float* log_lik, void* agg_out, int32_t* info, void* workspace,
                                     size_t workspace_bytes, void* stream);
hmm_status_t hmm_viterbi_dist_forward(int D, int64_t T_local, int64_t t_base, const float* log_pi,
                                      const float* log_A, const float* log_lik, const void* agg_all, int rank,
                                      int world, void* record_out, double* log_prob_partial, int32_t* info,
                                      void* workspace, size_t workspace_bytes, void* stream);
hmm_status_t hmm_viterbi_dist_finish(int D, int64_t T_local, int64_t t_base, const float* log_pi, const float* log_A,
                                     const float* log_lik, const void* records_all, int rank, int world,
                                     int32_t* path, int32_t* info, void* workspace, size_t workspace_bytes,
                                     void* stream);

/*
 * Split-phase scalar plumbing for a step that runs the smoother and Viterbi on the same partition with
 * merged collectives (paper_2102_05743_b200.dist.smooth_viterbi_dist), replacing a few dozen tiny
 * host-launched tensor ops per step by two launches; the smoother-only and Viterbi-only split steps use the
 * same pair (paper_2102_05743_b200.dist.smooth_dist / viterbi_dist).  All pointers are device memory; one
 * thread does the work, stream-ordered.  Any INPUT of hmm_dist_pack may be NULL (it contributes zeros);
 * any OUTPUT of hmm_dist_combine except `gathered` may be NULL (not written).  record16, packed8,
 * gathered, records_all and the doubles must be 8-byte aligned, the int32 words 4-byte aligned:
 * HMM_ERR_INVALID_VALUE otherwise, or for NULL packed8 / gathered, or world < 1.
 *   hmm_dist_pack: one rank's record as 8 doubles, packed8 = {the 16-byte Viterbi rank record
 *     (hmm_viterbi_dist_forward's record_out, bit-copied into doubles 0-1), log_z_partial,
 *     log_prob_partial, the four info codes (smoother reduce, smoother finish, Viterbi reduce, Viterbi
 *     forward) as doubles (exact)}.  The caller all-gathers packed8 into gathered[world][8], rank order.
 *   hmm_dist_combine: from gathered: records_all (16*world bytes, rank order, the input of
 *     hmm_viterbi_dist_finish), log_z = sum of the log_z partials and log_prob = sum of the log_prob
 *     partials, each added in rank order starting from 0.0 (log Z; Eq. 16-17), and the
 *     global info / vinfo: -1 if any rank reported -1 (bad input), else the smallest positive code (the
 *     first impossible global step + 1), else 0.
 */
hmm_status_t hmm_dist_pack(const void* record16, const double* log_z_partial, const double* log_prob_partial,
                           const int32_t* s_info_reduce, const int32_t* s_info_finish, const int32_t* v_info_reduce,
                           const int32_t* v_info_forward, double* packed8, void* stream);
hmm_status_t hmm_dist_combine(int world, const double* gathered, void* records_all, double* log_z,
                              double* log_prob, int32_t* info, int32_t* vinfo, void* stream);

/*
 * Profiling / introspection (not part of the compute path).
 *   hmm_debug_set_timers: for calls made later from the calling host thread, CTA phase timestamps
 *     (%globaltimer, ns) are written to device_buf[(b*G + c)*16 + i] (NULL disables).
 *   hmm_debug_plan: the launch plan for (op, D, T, B): out[0..7] = G (CTAs per sequence), R (steps per
 *     CTA; lane-streaming plan: steps per lane), S (steps per leaf / slice), chunk, K (chunks per CTA /
 *     slices per lane), kind (1 fused, 0 chunked, 2 lane-streaming), dynamic smem bytes, threads per
 *     CTA.  Returns 0 if unsupported.
 *   hmm_debug_force_path: for calls made later from the calling host thread, select the
 *     decomposition: 0 automatic (default); for 1 <= D <= 8 and B == 1: 1 lane-streaming (16-B
 *     aligned buffers required, else automatic), 2 resident/chunked; for 33 <= D <= 64: 3 keeps the
 *     sum-product leaf products on the FP32 CUDA cores instead of the tensor cores; for 9 <= D <= 32:
 *     4 forces the batch-parallel plan (one lane group per sequence running the Algorithm 1 / 4
 *     recursions, chosen automatically for large B; two warps per sequence running the forward and
 *     backward recursions from both ends while B fits one wave, else one warp), 5 forbids it (block
 *     scan), 6 forces the one-warp batch-parallel plan.  Test and profiling
 *     use only; the results agree within the stated tolerances whichever path runs.
 */
void hmm_debug_set_timers(unsigned long long* device_buf);
int hmm_debug_plan(int op, int D, int64_t T, int64_t B, int64_t* out);
void hmm_debug_force_path(int path);

#ifdef __cplusplus
}
#endif

#endif /* HMMSCAN_H */
