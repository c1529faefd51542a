/*
 * hmmgen.c — seeded synthetic HMM workloads shared by the oracle tests and the CUDA path.
 *
 * This module holds NONE of the method's arithmetic (no forward/backward, no Viterbi, no scan).
 * It only builds models and draws data, so both sides of a parity test consume bit-identical
 * fp32 inputs.  Recipes (DESIGN.md §"Input recipe"):
 *
 *   - Gilbert–Elliott (GE) channel, Eq. 22 of the paper verbatim, with the §VI
 *     parameters p0=.03 p1=.1 p2=.05 q0=.01 q1=.1 and a uniform prior.
 *   - Dense random model: rows of A ~ Dirichlet(1,...,1) (normalised Exp(1) variates), log taken in
 *     fp64, floored at -80, rounded to fp32; uniform prior; Gaussian emissions y_t = mu_{x_t} + N(0,1)
 *     with mu_d = d, log_lik_t(d) = -(y_t-d)^2/2 - log(2 pi)/2 (SURVEY.md §8(d) config ③/④).
 *   - Simulation (SPEC.md:362-366 contract): x_0 ~ pi, x_t ~ A[x_{t-1},:], y_t ~ emission row of x_t.
 *
 * Random numbers: a counter-based SplitMix64.  Uniform number k of stream `seed` is
 *   u(seed, k) = (splitmix64_mix(seed * 0x9E3779B97F4A7C15 + k + 1) >> 11) * 2^-53  in [0, 1).
 * Step t of a simulation uses counters 4t (state), 4t+1 (observation), 4t+2 and 4t+3 (Gaussian noise
 * / jitter, Box–Muller).  Being counter-based, any slice [t0, t1) can be generated independently.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

double hmmgen_uniform(uint64_t seed, uint64_t k) {
    uint64_t z = mix64(seed * 0x9E3779B97F4A7C15ULL + k + 1ULL);
    return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

/* Standard normal from counters (k, k+1) by Box–Muller (cosine branch). */
double hmmgen_normal(uint64_t seed, uint64_t k) {
    double u1 = hmmgen_uniform(seed, k);
    double u2 = hmmgen_uniform(seed, k + 1);
    if (u1 < 1e-300) u1 = 1e-300;
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925 * u2);
}

void hmmgen_uniform_fill(uint64_t seed, uint64_t k0, int64_t n, double* out) {
    for (int64_t i = 0; i < n; i++) out[i] = hmmgen_uniform(seed, k0 + (uint64_t)i);
}

/* Eq. 22 verbatim; row = x_{k-1}, column = x_k. */
void hmmgen_ge_model(double p0, double p1, double p2, double q0, double q1, double* Pi /*16*/,
                     double* O /*8*/, double* prior /*4*/) {
    const double P[16] = {
        (1 - p0) * (1 - p2), p0 * (1 - p2),       (1 - p0) * p2,       p0 * p2,
        p1 * (1 - p2),       (1 - p1) * (1 - p2), p1 * p2,             (1 - p1) * p2,
        (1 - p0) * p2,       p0 * p2,             (1 - p0) * (1 - p2), p0 * (1 - p2),
        p1 * p2,             (1 - p1) * p2,       p1 * (1 - p2),       (1 - p1) * (1 - p2)};
    const double E[8] = {1 - q0, q0, 1 - q1, q1, q0, 1 - q0, q1, 1 - q1};
    memcpy(Pi, P, sizeof(P));
    memcpy(O, E, sizeof(E));
    for (int i = 0; i < 4; i++) prior[i] = 0.25;
}

static inline int draw_categorical(const double* row, int n, double u) {
    double c = 0.0;
    for (int j = 0; j < n - 1; j++) {
        c += row[j];
        if (u < c) return j;
    }
    return n - 1;
}

/* Markov-chain simulation with a discrete emission matrix O[D,V] (row-stochastic). */
void hmmgen_simulate_discrete(int D, int V, const double* prior, const double* A, const double* O,
                              int64_t T, uint64_t seed, int32_t* states, int32_t* obs) {
    int x = 0;
    for (int64_t t = 0; t < T; t++) {
        double us = hmmgen_uniform(seed, 4 * (uint64_t)t);
        x = (t == 0) ? draw_categorical(prior, D, us) : draw_categorical(A + (size_t)x * D, D, us);
        states[t] = x;
        obs[t] = draw_categorical(O + (size_t)x * V, V, hmmgen_uniform(seed, 4 * (uint64_t)t + 1));
    }
}

/* log_lik[t,d] = (float) log O[d, y_t]  (O = p(y_k | x_k)). */
void hmmgen_loglik_discrete(int D, int V, const double* O, int64_t T, const int32_t* obs, float* log_lik) {
    double* lo = (double*)malloc(sizeof(double) * (size_t)D * V);
    for (int i = 0; i < D * V; i++) lo[i] = log(O[i]);
    for (int64_t t = 0; t < T; t++)
        for (int d = 0; d < D; d++) log_lik[t * D + d] = (float)lo[(size_t)d * V + obs[t]];
    free(lo);
}

/* Dense model: A rows ~ Dirichlet(1): normalised -log(u) variates; logs floored at -80, fp32. */
void hmmgen_dense_model(int D, uint64_t seed, float* log_pi, float* log_A, double* A_out /*nullable*/) {
    double* row = (double*)malloc(sizeof(double) * D);
    for (int i = 0; i < D; i++) {
        double s = 0.0;
        for (int j = 0; j < D; j++) {
            double u = hmmgen_uniform(seed, (uint64_t)i * D + j);
            if (u < 1e-300) u = 1e-300;
            row[j] = -log(u);
            s += row[j];
        }
        for (int j = 0; j < D; j++) {
            double p = row[j] / s;
            double lp = log(p);
            if (lp < -80.0) lp = -80.0;
            log_A[i * D + j] = (float)lp;
            if (A_out) A_out[i * D + j] = p;
        }
        log_pi[i] = (float)(-log((double)D));
    }
    free(row);
}

/* Simulate states from (pi, A) given in fp32 log form, then Gaussian emissions mu_d = d. */
void hmmgen_simulate_gaussian(int D, const float* log_pi, const float* log_A, int64_t T, uint64_t seed,
                              int32_t* states, float* log_lik) {
    double* P = (double*)malloc(sizeof(double) * (size_t)D * D);
    double* pr = (double*)malloc(sizeof(double) * D);
    double s0 = 0.0;
    for (int i = 0; i < D; i++) { pr[i] = exp((double)log_pi[i]); s0 += pr[i]; }
    for (int i = 0; i < D; i++) pr[i] /= s0;
    for (int i = 0; i < D; i++) {
        double s = 0.0;
        for (int j = 0; j < D; j++) { P[i * D + j] = exp((double)log_A[i * D + j]); s += P[i * D + j]; }
        for (int j = 0; j < D; j++) P[i * D + j] /= s;
    }
    const double half_log_2pi = 0.91893853320467274178;
    int x = 0;
    for (int64_t t = 0; t < T; t++) {
        double us = hmmgen_uniform(seed, 4 * (uint64_t)t);
        x = (t == 0) ? draw_categorical(pr, D, us) : draw_categorical(P + (size_t)x * D, D, us);
        if (states) states[t] = x;
        double y = (double)x + hmmgen_normal(seed, 4 * (uint64_t)t + 2);
        for (int d = 0; d < D; d++) {
            double r = y - (double)d;
            log_lik[t * D + d] = (float)(-0.5 * r * r - half_log_2pi);
        }
    }
    free(P);
    free(pr);
}

/* log_lik += sigma * N(0,1), per element counter 2*(t*D+d) in stream `seed` (jittered GE copies). */
void hmmgen_jitter(int D, int64_t T, float* log_lik, double sigma, uint64_t seed) {
    for (int64_t t = 0; t < T; t++)
        for (int d = 0; d < D; d++) {
            uint64_t k = 2 * ((uint64_t)t * D + d);
            log_lik[t * D + d] = (float)((double)log_lik[t * D + d] + sigma * hmmgen_normal(seed, k));
        }
}

/* i.i.d. N(mu, sigma^2) fill (secondary dense workload, random potentials). */
void hmmgen_normal_fill(int64_t n, float* out, double mu, double sigma, uint64_t seed) {
    for (int64_t i = 0; i < n; i++) out[i] = (float)(mu + sigma * hmmgen_normal(seed, 2 * (uint64_t)i));
}
