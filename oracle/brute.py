"""Brute-force enumeration over all D^T state sequences — TEST INFRASTRUCTURE ONLY.

Eq. 1 (partition function Z), Eq. 2 (marginals), Eq. 3 / Eq. 17
(max / MAP) written out literally over the potentials of Eq. 5
(PAPER.md:102-108): psi_1(x_1) = p(y_1|x_1) p(x_1), psi_k(x_{k-1},x_k) = p(y_k|x_k) p(x_k|x_{k-1}).
Independent of ``hmm_oracle.c`` (different language, no recursion) so it can pin it.
MAP ties: lexicographically smallest sequence.
"""
from __future__ import annotations

import itertools

import numpy as np

MAX_SEQUENCES = 2_000_000


def _all_sequences(D: int, T: int) -> np.ndarray:
    if D ** T > MAX_SEQUENCES:
        raise ValueError(f"D^T = {D}^{T} exceeds the brute-force guard {MAX_SEQUENCES}")
    # itertools.product enumerates in lexicographic order.
    return np.array(list(itertools.product(range(D), repeat=T)), dtype=np.int64).reshape(-1, T)


def joint_log_weights(log_pi, log_A, log_lik, X: np.ndarray) -> np.ndarray:
    """log[psi_1(x_1) prod_{t>=2} psi_t(x_{t-1}, x_t)] for every row of X (Eq. 6)."""
    lp = np.asarray(log_pi, np.float64); la = np.asarray(log_A, np.float64); ll = np.asarray(log_lik, np.float64)
    T = X.shape[1]
    w = lp[X[:, 0]] + ll[0, X[:, 0]]
    for t in range(1, T):
        w = w + la[X[:, t - 1], X[:, t]] + ll[t, X[:, t]]
    return w


def _logsumexp(w: np.ndarray) -> float:
    m = np.max(w)
    if m == -np.inf:
        return -np.inf
    return float(m + np.log(np.sum(np.exp(w - m))))


def smooth(log_pi, log_A, log_lik):
    """Returns dict(log_z, smoothed [T,D], filtered [T,D]) by enumeration.

    filtered[t] = p(x_t | y_0..y_t) is the last-position marginal of the model truncated at t
    (the forward pass is filtering).
    """
    ll = np.asarray(log_lik, np.float64)
    T, D = ll.shape
    X = _all_sequences(D, T)
    w = joint_log_weights(log_pi, log_A, ll, X)
    lz = _logsumexp(w)
    p = np.exp(w - lz)
    sm = np.zeros((T, D))
    for t in range(T):
        sm[t] = np.bincount(X[:, t], weights=p, minlength=D)
    filt = np.zeros((T, D))
    for t in range(T):
        Xt = _all_sequences(D, t + 1)
        wt = joint_log_weights(log_pi, log_A, ll[: t + 1], Xt)
        pt = np.exp(wt - _logsumexp(wt))
        filt[t] = np.bincount(Xt[:, t], weights=pt, minlength=D)
    return dict(log_z=lz, smoothed=sm, filtered=filt)


def pair_stats(log_pi, log_A, log_lik):
    """Baum-Welch E-step statistics by enumeration: xi_sum[i,j] = sum_{t>=1} p(x_{t-1}=i, x_t=j | y)
    and gamma_sum[d] = sum_t p(x_t=d | y) over the normalised joint weights of Eq. 6."""
    ll = np.asarray(log_lik, np.float64)
    T, D = ll.shape
    X = _all_sequences(D, T)
    w = joint_log_weights(log_pi, log_A, ll, X)
    p = np.exp(w - _logsumexp(w))
    xi = np.zeros((D, D))
    for t in range(1, T):
        np.add.at(xi, (X[:, t - 1], X[:, t]), p)
    g = np.zeros(D)
    for t in range(T):
        g += np.bincount(X[:, t], weights=p, minlength=D)
    return dict(xi_sum=xi, gamma_sum=g)


def viterbi(log_pi, log_A, log_lik, tie_tol: float = 1e-9):
    """MAP sequence by enumeration; among sequences within tie_tol of the best, the lexicographically
    smallest.  Returns dict(path, log_prob, gap) with gap = best - second best distinct-sequence weight."""
    ll = np.asarray(log_lik, np.float64)
    T, D = ll.shape
    X = _all_sequences(D, T)
    w = joint_log_weights(log_pi, log_A, ll, X)
    best = np.max(w)
    cand = np.nonzero(w >= best - tie_tol)[0]
    k = int(cand[0])  # lexicographic order of enumeration
    ws = np.sort(w)[::-1]
    gap = float(ws[0] - ws[1]) if len(ws) > 1 else np.inf
    return dict(path=X[k].astype(np.int32), log_prob=float(best), gap=gap)


def max_marginals(log_pi, log_A, log_lik):
    """Eq. 3: p*(x_k) = max over all other variables (log domain)."""
    ll = np.asarray(log_lik, np.float64)
    T, D = ll.shape
    X = _all_sequences(D, T)
    w = joint_log_weights(log_pi, log_A, ll, X)
    out = np.full((T, D), -np.inf)
    for t in range(T):
        for d in range(D):
            sel = X[:, t] == d
            if sel.any():
                out[t, d] = np.max(w[sel])
    return out
