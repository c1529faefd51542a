/*
 * hmm_oracle.c — plain, slow, sequential fp64 reference for the HMM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header, table or constant with
 * the CUDA path (paper_2102_05743_b200/); both sides only share the seeded input generators in
 * workloads/.
 *
 * What it computes (the plain definitions the parallel method reaches "algebraically"):
 *
 *   oracle_smooth   — Algorithm 1, the classical sum-product forward/backward
 *                     pass over the potentials of Eq. 5, with the usual per-step
 *                     normalisation (scaling) so fp64 does not underflow; marginals by Eq. 10 / Eq. 14
 *                     (PAPER.md:147-154, 381-385); filtered = normalised forward potential;
 *                     log Z = log of the partition function of Eq. 1.
 *   oracle_viterbi  — Algorithm 4, in the log domain, smallest-index ties
 *                     (SURVEY.md §8(c) reading 5).
 *   oracle_max_marginals — Lemma 3 recursions: log psi~f_k (= V_k) and log psi~b_k;
 *                     their sum is the max-marginal of Eq. 3; used for gap / tie analysis
 *                     and the Theorem 4 invariant.  Diagnostics, not outputs.
 *   oracle_joint_weight — log of psi_1(x_1) prod psi_t(x_{t-1},x_t) (Eq. 6).
 *   oracle_max_marginal_gap / oracle_joint_weight_diff — the same quantities in O(T) memory / without
 *                     cancellation, for checking full-size (T = 1e8) paths.
 *
 * Conventions: 0-based t; log_A[i*D+j] = log p(x_t=j | x_{t-1}=i);
 * log_lik[t*D+d] = log p(y_t | x_t=d); inputs are fp32, promoted to fp64 on read.
 * info = 0 ok; t+1 for the first t at which no state sequence is consistent with the evidence
 * (zero forward mass / all V_t = -inf); -1 if a NaN or +inf input is seen.
 *
 * Parity pins for this file live in tests/test_oracle_pins.py (brute force over D^T sequences,
 * closed forms, invariants, and the fixtures in tests/golden/).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static int has_bad(const float* x, int64_t n) {
    for (int64_t i = 0; i < n; i++)
        if (isnan(x[i]) || (isinf(x[i]) && x[i] > 0)) return 1;
    return 0;
}

/* Algorithm 1 with per-step normalisation.
 * Outputs: filtered[T*D], smoothed[T*D] (either may be NULL), log_z_fwd, log_z_bwd (nullable).   */
int oracle_smooth(int D, int64_t T, const float* log_pi, const float* log_A, const float* log_lik,
                  double* filtered, double* smoothed, double* log_z_fwd, double* log_z_bwd, int64_t* info) {
    *info = 0;
    if (has_bad(log_pi, D) || has_bad(log_A, (int64_t)D * D) || has_bad(log_lik, T * D)) { *info = -1; return 0; }
    double* A = (double*)malloc(sizeof(double) * D * D);
    double* pi = (double*)malloc(sizeof(double) * D);
    double* alpha = (double*)malloc(sizeof(double) * (size_t)T * D); /* normalised forward potentials */
    double* beta = (double*)malloc(sizeof(double) * (size_t)T * D);  /* normalised backward potentials */
    double* l = (double*)malloc(sizeof(double) * D);
    double* m = (double*)malloc(sizeof(double) * T);                 /* per-step max log-likelihood */
    for (int i = 0; i < D * D; i++) A[i] = exp((double)log_A[i]);
    for (int i = 0; i < D; i++) pi[i] = exp((double)log_pi[i]);

    /* Per-step likelihood l_t(d) = exp(log_lik_t(d) - m_t), m_t = max_d log_lik_t(d). */
#define LIK(t)                                                                   \
    do {                                                                         \
        double mx = -INFINITY;                                                   \
        for (int d = 0; d < D; d++) if ((double)log_lik[(t) * D + d] > mx) mx = log_lik[(t) * D + d]; \
        m[t] = mx;                                                               \
        for (int d = 0; d < D; d++)                                              \
            l[d] = (mx == -INFINITY) ? 0.0 : exp((double)log_lik[(t) * D + d] - mx); \
    } while (0)

    /* Forward pass: psi^f_{1,1} = psi_1 (Alg 1 line 2); psi^f_{1,k} = sum_{x_{k-1}} psi^f psi_{k-1,k} (line 4). */
    double lz = 0.0;
    int64_t bad_t = -1;
    for (int64_t t = 0; t < T; t++) {
        LIK(t);
        double* a = alpha + (size_t)t * D;
        if (t == 0) {
            for (int j = 0; j < D; j++) a[j] = pi[j] * l[j];                 /* psi_1 = p(y_1|x_1) p(x_1) */
        } else {
            const double* ap = alpha + (size_t)(t - 1) * D;
            for (int j = 0; j < D; j++) {
                double s = 0.0;
                for (int i = 0; i < D; i++) s += ap[i] * A[i * D + j];     /* sum_{x_{k-1}} psi^f * p(x_k|x_{k-1}) */
                a[j] = s * l[j];                                            /* * p(y_k|x_k) */
            }
        }
        double c = 0.0;
        for (int j = 0; j < D; j++) c += a[j];
        if (!(c > 0.0)) { bad_t = t; break; }
        for (int j = 0; j < D; j++) a[j] /= c;
        lz += log(c) + m[t];
    }
    if (bad_t >= 0) {
        *info = bad_t + 1;
        if (filtered) for (int64_t i = 0; i < T * D; i++) filtered[i] = NAN;
        if (smoothed) for (int64_t i = 0; i < T * D; i++) smoothed[i] = NAN;
        if (log_z_fwd) *log_z_fwd = NAN;
        if (log_z_bwd) *log_z_bwd = NAN;
        free(A); free(pi); free(alpha); free(beta); free(l); free(m);
        return 0;
    }
    if (log_z_fwd) *log_z_fwd = lz;

    /* Backward pass: psi^b_{T,T} = 1 (Alg 1 line 7); psi^b_{k,T} = sum_{x_{k+1}} psi_{k,k+1} psi^b_{k+1,T} (line 9). */
    double lzb = 0.0;
    for (int d = 0; d < D; d++) beta[(size_t)(T - 1) * D + d] = 1.0;
    for (int64_t t = T - 2; t >= 0; t--) {
        LIK(t + 1);
        const double* bn = beta + (size_t)(t + 1) * D;
        double* b = beta + (size_t)t * D;
        double s = 0.0;
        for (int i = 0; i < D; i++) {
            double acc = 0.0;
            for (int j = 0; j < D; j++) acc += A[i * D + j] * l[j] * bn[j];  /* psi_{k,k+1}(x_k,x_{k+1}) psi^b */
            b[i] = acc;
            s += acc;
        }
        for (int i = 0; i < D; i++) b[i] /= s;
        lzb += log(s) + m[t + 1];
    }
    LIK(0);
    {
        double s = 0.0;
        for (int d = 0; d < D; d++) s += pi[d] * l[d] * beta[d];
        lzb += log(s) + m[0];
    }
    if (log_z_bwd) *log_z_bwd = lzb;

    /* Marginals, Eq. 10 / Eq. 14: p(x_k) = psi^f psi^b / Z_k. */
    for (int64_t t = 0; t < T; t++) {
        const double* a = alpha + (size_t)t * D;
        const double* b = beta + (size_t)t * D;
        if (filtered) for (int d = 0; d < D; d++) filtered[t * D + d] = a[d];
        if (smoothed) {
            double z = 0.0;
            for (int d = 0; d < D; d++) z += a[d] * b[d];
            for (int d = 0; d < D; d++) smoothed[t * D + d] = a[d] * b[d] / z;
        }
    }
#undef LIK
    free(A); free(pi); free(alpha); free(beta); free(l); free(m);
    return 0;
}

/* Algorithm 1 again, keeping only the rows at the sorted sample steps ts[0..ns) (O(ns) memory, for
 * checking full-size runs at sampled outputs).  Same recursions and normalisation as oracle_smooth:
 * the forward potentials are kept at the sampled steps during the forward pass, the backward
 * potentials during the backward pass, and Eq. 14 combines them.  filtered_s / smoothed_s are
 * [ns*D]; log_z is the forward-pass log Z.                                                          */
int oracle_smooth_sampled(int D, int64_t T, const float* log_pi, const float* log_A, const float* log_lik,
                          const int64_t* ts, int64_t ns, double* filtered_s, double* smoothed_s, double* log_z,
                          int64_t* info) {
    *info = 0;
    if (has_bad(log_pi, D) || has_bad(log_A, (int64_t)D * D) || has_bad(log_lik, T * D)) { *info = -1; return 0; }
    double A[64 * 64], pi[64], a[64], an[64], b[64], bn[64], l[64];
    if (D > 64) return 1;
    for (int i = 0; i < D * D; i++) A[i] = exp((double)log_A[i]);
    for (int i = 0; i < D; i++) pi[i] = exp((double)log_pi[i]);
    double* bs = (double*)malloc(sizeof(double) * (size_t)(ns > 0 ? ns : 1) * D);
#define LIKS(t, mx)                                                              \
    do {                                                                         \
        mx = -INFINITY;                                                          \
        for (int d = 0; d < D; d++) if ((double)log_lik[(t) * D + d] > mx) mx = log_lik[(t) * D + d]; \
        for (int d = 0; d < D; d++)                                              \
            l[d] = (mx == -INFINITY) ? 0.0 : exp((double)log_lik[(t) * D + d] - mx); \
    } while (0)
    /* forward (Alg 1 lines 2-4), normalised */
    double lz = 0.0, mx;
    int64_t q = 0;
    for (int64_t t = 0; t < T; t++) {
        LIKS(t, mx);
        if (t == 0) {
            for (int j = 0; j < D; j++) an[j] = pi[j] * l[j];
        } else {
            for (int j = 0; j < D; j++) {
                double s = 0.0;
                for (int i = 0; i < D; i++) s += a[i] * A[i * D + j];
                an[j] = s * l[j];
            }
        }
        double c = 0.0;
        for (int j = 0; j < D; j++) c += an[j];
        if (!(c > 0.0)) { *info = t + 1; free(bs); *log_z = NAN; return 0; }
        for (int j = 0; j < D; j++) a[j] = an[j] / c;
        lz += log(c) + mx;
        while (q < ns && ts[q] == t) {
            for (int j = 0; j < D; j++) filtered_s[q * D + j] = a[j];
            q++;
        }
    }
    *log_z = lz;
    /* backward (Alg 1 lines 7-9), normalised like oracle_smooth */
    for (int d = 0; d < D; d++) b[d] = 1.0;
    q = ns - 1;
    for (int64_t t = T - 1; t >= 0; t--) {
        if (t < T - 1) {
            LIKS(t + 1, mx);
            double s = 0.0;
            for (int i = 0; i < D; i++) {
                double acc = 0.0;
                for (int j = 0; j < D; j++) acc += A[i * D + j] * l[j] * b[j];
                bn[i] = acc;
                s += acc;
            }
            for (int i = 0; i < D; i++) b[i] = bn[i] / s;
        }
        while (q >= 0 && ts[q] == t) {
            for (int j = 0; j < D; j++) bs[q * D + j] = b[j];
            q--;
        }
    }
    /* Eq. 14 at the sampled steps */
    for (int64_t k = 0; k < ns; k++) {
        double z = 0.0;
        for (int d = 0; d < D; d++) z += filtered_s[k * D + d] * bs[k * D + d];
        for (int d = 0; d < D; d++) smoothed_s[k * D + d] = filtered_s[k * D + d] * bs[k * D + d] / z;
    }
#undef LIKS
    free(bs);
    return 0;
}

/* Baum-Welch expectation statistics ("in expectation step, BWA uses the forward-backward
 * algorithm"): with the normalised forward potentials alpha_t and backward potentials beta_t of
 * Algorithm 1 (as in oracle_smooth), the pairwise posterior of Eq. 6's factorisation
 *   xi_t(i,j) = p(x_{t-1}=i, x_t=j | y) = alpha_{t-1}(i) A(i,j) l_t(j) beta_t(j) / sum_{i,j}(same)
 * summed over t = 1..T-1 into xi_sum[D*D], and the occupancies gamma_sum[d] = sum_t p(x_t=d | y)
 * (Eq. 14).  log_z as oracle_smooth's forward pass.                                                   */
int oracle_smooth_stats(int D, int64_t T, const float* log_pi, const float* log_A, const float* log_lik,
                        double* xi_sum, double* gamma_sum, double* log_z, int64_t* info) {
    double* sm = (double*)malloc(sizeof(double) * (size_t)T * D);
    double* fl = (double*)malloc(sizeof(double) * (size_t)T * D);
    double lzb;
    oracle_smooth(D, T, log_pi, log_A, log_lik, fl, sm, log_z, &lzb, info);
    for (int i = 0; i < D * D; i++) xi_sum[i] = 0.0;
    for (int i = 0; i < D; i++) gamma_sum[i] = 0.0;
    if (*info != 0) { free(sm); free(fl); return 0; }
    /* smoothed_t = alpha_t beta_t / Z_t  =>  beta_t(j) proportional to smoothed_t(j) / alpha_t(j) where
     * alpha_t(j) > 0; recompute beta directly instead (Alg 1 lines 7-9) to stay on the definition. */
    double* A = (double*)malloc(sizeof(double) * D * D);
    double* beta = (double*)malloc(sizeof(double) * (size_t)T * D);
    double* l = (double*)malloc(sizeof(double) * D);
    for (int i = 0; i < D * D; i++) A[i] = exp((double)log_A[i]);
    for (int d = 0; d < D; d++) beta[(size_t)(T - 1) * D + d] = 1.0;
    for (int64_t t = T - 2; t >= 0; t--) {
        double mx = -INFINITY;
        for (int d = 0; d < D; d++) if ((double)log_lik[(t + 1) * D + d] > mx) mx = log_lik[(t + 1) * D + d];
        for (int d = 0; d < D; d++) l[d] = (mx == -INFINITY) ? 0.0 : exp((double)log_lik[(t + 1) * D + d] - mx);
        double s = 0.0;
        for (int i = 0; i < D; i++) {
            double acc = 0.0;
            for (int j = 0; j < D; j++) acc += A[i * D + j] * l[j] * beta[(size_t)(t + 1) * D + j];
            beta[(size_t)t * D + i] = acc;
            s += acc;
        }
        for (int i = 0; i < D; i++) beta[(size_t)t * D + i] /= s;
    }
    double* x = (double*)malloc(sizeof(double) * D * D);
    for (int64_t t = 1; t < T; t++) {
        double mx = -INFINITY;
        for (int d = 0; d < D; d++) if ((double)log_lik[t * D + d] > mx) mx = log_lik[t * D + d];
        for (int d = 0; d < D; d++) l[d] = (mx == -INFINITY) ? 0.0 : exp((double)log_lik[t * D + d] - mx);
        double z = 0.0;
        for (int i = 0; i < D; i++)
            for (int j = 0; j < D; j++) {
                x[i * D + j] = fl[(size_t)(t - 1) * D + i] * A[i * D + j] * l[j] * beta[(size_t)t * D + j];
                z += x[i * D + j];
            }
        for (int i = 0; i < D * D; i++) xi_sum[i] += x[i] / z;
    }
    for (int64_t t = 0; t < T; t++)
        for (int d = 0; d < D; d++) gamma_sum[d] += sm[(size_t)t * D + d];
    free(A); free(beta); free(l); free(x); free(sm); free(fl);
    return 0;
}

/* Algorithm 4 in the log domain.  path[T] int32, log_prob = max_x V_T(x). */
int oracle_viterbi(int D, int64_t T, const float* log_pi, const float* log_A, const float* log_lik,
                   int32_t* path, double* log_prob, int64_t* info) {
    *info = 0;
    if (has_bad(log_pi, D) || has_bad(log_A, (int64_t)D * D) || has_bad(log_lik, T * D)) { *info = -1; return 0; }
    double* V = (double*)malloc(sizeof(double) * D);
    double* Vn = (double*)malloc(sizeof(double) * D);
    uint8_t* u = (uint8_t*)malloc((size_t)T * D); /* u_{t-1}(x_t) stored at u[t*D + x_t], t >= 1 */
    /* V_1(x_1) = psi_1(x_1)  (line 2) */
    for (int j = 0; j < D; j++) V[j] = (double)log_pi[j] + (double)log_lik[j];
    int64_t bad_t = -1;
    {
        double mx = -INFINITY;
        for (int j = 0; j < D; j++) if (V[j] > mx) mx = V[j];
        if (mx == -INFINITY) bad_t = 0;
    }
    for (int64_t t = 1; t < T && bad_t < 0; t++) {
        double mx = -INFINITY;
        for (int j = 0; j < D; j++) {
            /* V_k(x_k) = max_{x_{k-1}} [psi_k(x_{k-1},x_k) V_{k-1}(x_{k-1})]   (line 4)
             * u_{k-1}(x_k) = argmax, smallest index on ties                     (line 5) */
            double best = -INFINITY;
            int arg = 0;
            for (int i = 0; i < D; i++) {
                double s = V[i] + (double)log_A[i * D + j];
                if (s > best) { best = s; arg = i; }
            }
            Vn[j] = best + (double)log_lik[t * D + j];
            u[t * D + j] = (uint8_t)arg;
            if (Vn[j] > mx) mx = Vn[j];
        }
        memcpy(V, Vn, sizeof(double) * D);
        if (mx == -INFINITY) bad_t = t;
    }
    if (bad_t >= 0) {
        *info = bad_t + 1;
        for (int64_t t = 0; t < T; t++) path[t] = -1;
        *log_prob = NAN;
        free(V); free(Vn); free(u);
        return 0;
    }
    /* x*_T = argmax V_T (line 8); x*_{k-1} = u_{k-1}(x*_k) (lines 9-11) */
    int x = 0;
    double best = -INFINITY;
    for (int j = 0; j < D; j++) if (V[j] > best) { best = V[j]; x = j; }
    *log_prob = best;
    path[T - 1] = x;
    for (int64_t t = T - 1; t >= 1; t--) {
        x = u[t * D + x];
        path[t - 1] = x;
    }
    free(V); free(Vn); free(u);
    return 0;
}

/* Lemma 3 in the log domain:
 *   fwd[t] = log psi~f_t  (= V_t of Alg 4),  bwd[t] = log psi~b_t with bwd[T-1] = 0,
 *   score[t*D+x] = fwd + bwd (log max-marginal, Eq. 3), gap[t] = best - second best score at t
 *   (+inf when D == 1).  Any of the outputs may be NULL.                                          */
int oracle_max_marginals(int D, int64_t T, const float* log_pi, const float* log_A, const float* log_lik,
                         double* score, double* gap) {
    double* f = (double*)malloc(sizeof(double) * (size_t)T * D);
    double* b = (double*)malloc(sizeof(double) * (size_t)T * D);
    for (int j = 0; j < D; j++) f[j] = (double)log_pi[j] + (double)log_lik[j];
    for (int64_t t = 1; t < T; t++)
        for (int j = 0; j < D; j++) {
            double best = -INFINITY;
            for (int i = 0; i < D; i++) {
                double s = f[(t - 1) * D + i] + (double)log_A[i * D + j];
                if (s > best) best = s;
            }
            f[t * D + j] = best + (double)log_lik[t * D + j];
        }
    for (int i = 0; i < D; i++) b[(T - 1) * D + i] = 0.0;
    for (int64_t t = T - 2; t >= 0; t--)
        for (int i = 0; i < D; i++) {
            double best = -INFINITY;
            for (int j = 0; j < D; j++) {
                double s = (double)log_A[i * D + j] + (double)log_lik[(t + 1) * D + j] + b[(t + 1) * D + j];
                if (s > best) best = s;
            }
            b[t * D + i] = best;
        }
    for (int64_t t = 0; t < T; t++) {
        double b1 = -INFINITY, b2 = -INFINITY;
        for (int x = 0; x < D; x++) {
            double s = f[t * D + x] + b[t * D + x];
            if (score) score[t * D + x] = s;
            if (s > b1) { b2 = b1; b1 = s; } else if (s > b2) b2 = s;
        }
        if (gap) gap[t] = (D == 1) ? INFINITY : b1 - b2;
    }
    free(f); free(b);
    return 0;
}

/* The per-step max-marginal gap of oracle_max_marginals (Lemma 3; Eq. 3) in O(T) memory
 * for full-size checks (T = 1e8): gap32[t] = (float)(best - second best of fwd[t] + bwd[t]).  Same
 * recursions, operand order and tie loop as oracle_max_marginals, so the values are bitwise the ones it
 * computes; only the storage differs: the forward values are kept at every K-th step (checkpoints) and
 * recomputed one block at a time while the backward recursion runs right to left.                       */
int oracle_max_marginal_gap(int D, int64_t T, const float* log_pi, const float* log_A, const float* log_lik,
                            float* gap32) {
    const int64_t K = 4096;
    const int64_t nb = (T + K - 1) / K;
    double* ck = (double*)malloc(sizeof(double) * (size_t)nb * D); /* fwd at t = b*K */
    double* fb = (double*)malloc(sizeof(double) * (size_t)K * D);  /* fwd over one block */
    double *f = (double*)malloc(sizeof(double) * D), *fn = (double*)malloc(sizeof(double) * D);
    double *b = (double*)malloc(sizeof(double) * D), *bn = (double*)malloc(sizeof(double) * D);
    if (!ck || !fb || !f || !fn || !b || !bn) { free(ck); free(fb); free(f); free(fn); free(b); free(bn); return 1; }
    /* forward: psi~f (Lemma 3), checkpointed */
    for (int j = 0; j < D; j++) f[j] = (double)log_pi[j] + (double)log_lik[j];
    for (int64_t t = 0; t < T; t++) {
        if (t > 0) {
            for (int j = 0; j < D; j++) {
                double best = -INFINITY;
                for (int i = 0; i < D; i++) {
                    double s = f[i] + (double)log_A[i * D + j];
                    if (s > best) best = s;
                }
                fn[j] = best + (double)log_lik[t * D + j];
            }
            memcpy(f, fn, sizeof(double) * D);
        }
        if (t % K == 0) memcpy(ck + (size_t)(t / K) * D, f, sizeof(double) * D);
    }
    /* backward: psi~b, one block at a time from the right, with the block's fwd recomputed */
    for (int i = 0; i < D; i++) b[i] = 0.0;
    for (int64_t blk = nb - 1; blk >= 0; blk--) {
        const int64_t t0 = blk * K, t1 = (t0 + K < T) ? t0 + K : T;
        memcpy(fb, ck + (size_t)blk * D, sizeof(double) * D);
        for (int64_t t = t0 + 1; t < t1; t++) {
            const double* fp = fb + (size_t)(t - 1 - t0) * D;
            for (int j = 0; j < D; j++) {
                double best = -INFINITY;
                for (int i = 0; i < D; i++) {
                    double s = fp[i] + (double)log_A[i * D + j];
                    if (s > best) best = s;
                }
                fb[(size_t)(t - t0) * D + j] = best + (double)log_lik[t * D + j];
            }
        }
        for (int64_t t = t1 - 1; t >= t0; t--) {
            if (t < T - 1) {
                for (int i = 0; i < D; i++) {
                    double best = -INFINITY;
                    for (int j = 0; j < D; j++) {
                        double s = (double)log_A[i * D + j] + (double)log_lik[(t + 1) * D + j] + b[j];
                        if (s > best) best = s;
                    }
                    bn[i] = best;
                }
                memcpy(b, bn, sizeof(double) * D);
            }
            double b1 = -INFINITY, b2 = -INFINITY;
            for (int x = 0; x < D; x++) {
                double s = fb[(size_t)(t - t0) * D + x] + b[x];
                if (s > b1) { b2 = b1; b1 = s; } else if (s > b2) b2 = s;
            }
            gap32[t] = (float)((D == 1) ? INFINITY : b1 - b2);
        }
    }
    free(ck); free(fb); free(f); free(fn); free(b); free(bn);
    return 0;
}

/* Difference of the joint log-weights (Eq. 6) of two state sequences a and b,
 * log w(a) - log w(b), summed only over the terms that differ (the prior/evidence term at t and the
 * transition term into t, wherever a or its predecessor differs from b).  Equal to
 * oracle_joint_weight(a) - oracle_joint_weight(b) but without cancelling two ~1e7-nat sums, so a loss of
 * 1e-6 nats is resolvable at T = 1e8.                                                                    */
double oracle_joint_weight_diff(int D, int64_t T, const float* log_pi, const float* log_A, const float* log_lik,
                                const int32_t* a, const int32_t* b) {
    double d = 0.0;
    for (int64_t t = 0; t < T; t++) {
        const int diff_here = a[t] != b[t];
        const int diff_prev = t > 0 && a[t - 1] != b[t - 1];
        if (!diff_here && !diff_prev) continue;
        double wa, wb;
        if (t == 0) {
            wa = (double)log_pi[a[0]] + (double)log_lik[a[0]];
            wb = (double)log_pi[b[0]] + (double)log_lik[b[0]];
        } else {
            wa = (double)log_A[a[t - 1] * D + a[t]] + (double)log_lik[t * D + a[t]];
            wb = (double)log_A[b[t - 1] * D + b[t]] + (double)log_lik[t * D + b[t]];
        }
        d += wa - wb;
    }
    return d;
}

/* log psi_1(x_1) + sum_t log psi_t(x_{t-1}, x_t)  (Eq. 6; Eq. 16 joint). */
double oracle_joint_weight(int D, int64_t T, const float* log_pi, const float* log_A, const float* log_lik,
                           const int32_t* path) {
    double w = (double)log_pi[path[0]] + (double)log_lik[path[0]];
    for (int64_t t = 1; t < T; t++)
        w += (double)log_A[path[t - 1] * D + path[t]] + (double)log_lik[t * D + path[t]];
    return w;
}

/* ---- batched: B independent sequences sharing (log_pi, log_A), spread over host threads ---- */
typedef struct {
    int D; int64_t T; int64_t b0, b1; int op;
    const float *log_pi, *log_A, *log_lik;
    double *filtered, *smoothed, *lz, *lzb, *log_prob; int32_t* path; int64_t* info;
} job_t;

static void* run_job(void* p) {
    job_t* j = (job_t*)p;
    for (int64_t b = j->b0; b < j->b1; b++) {
        const float* ll = j->log_lik + (size_t)b * j->T * j->D;
        if (j->op == 0)
            oracle_smooth(j->D, j->T, j->log_pi, j->log_A, ll,
                          j->filtered ? j->filtered + (size_t)b * j->T * j->D : NULL,
                          j->smoothed ? j->smoothed + (size_t)b * j->T * j->D : NULL,
                          j->lz + b, j->lzb ? j->lzb + b : NULL, j->info + b);
        else
            oracle_viterbi(j->D, j->T, j->log_pi, j->log_A, ll, j->path + (size_t)b * j->T,
                           j->log_prob + b, j->info + b);
    }
    return NULL;
}

static int run_batched(job_t base, int64_t B, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > B) nthreads = (int)B;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
    job_t* jobs = (job_t*)malloc(sizeof(job_t) * nthreads);
    for (int k = 0; k < nthreads; k++) {
        jobs[k] = base;
        jobs[k].b0 = B * k / nthreads;
        jobs[k].b1 = B * (k + 1) / nthreads;
        pthread_create(&th[k], NULL, run_job, &jobs[k]);
    }
    for (int k = 0; k < nthreads; k++) pthread_join(th[k], NULL);
    free(th); free(jobs);
    return 0;
}

int oracle_smooth_batched(int D, int64_t T, int64_t B, const float* log_pi, const float* log_A,
                          const float* log_lik, double* filtered, double* smoothed, double* log_z,
                          double* log_z_bwd, int64_t* info, int nthreads) {
    job_t j;
    memset(&j, 0, sizeof(j));
    j.D = D; j.T = T; j.op = 0; j.log_pi = log_pi; j.log_A = log_A; j.log_lik = log_lik;
    j.filtered = filtered; j.smoothed = smoothed; j.lz = log_z; j.lzb = log_z_bwd; j.info = info;
    return run_batched(j, B, nthreads);
}

int oracle_viterbi_batched(int D, int64_t T, int64_t B, const float* log_pi, const float* log_A,
                           const float* log_lik, int32_t* path, double* log_prob, int64_t* info, int nthreads) {
    job_t j;
    memset(&j, 0, sizeof(j));
    j.D = D; j.T = T; j.op = 1; j.log_pi = log_pi; j.log_A = log_A; j.log_lik = log_lik;
    j.path = path; j.log_prob = log_prob; j.info = info;
    return run_batched(j, B, nthreads);
}
