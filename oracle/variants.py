"""fp64 oracle of the paper-faithful Viterbi variants — TEST INFRASTRUCTURE ONLY.

Only ``tests/`` may import this module; it shares no code with the CUDA path.

* ``viterbi_maxproduct`` — Algorithm 5: the forward max-product scan gives the
  maximum forward potentials psi~f_k (Proposition 2), the reversed scan the maximum
  backward potentials psi~b_k (Proposition 3); both equal the Lemma 3 recursions
  (PAPER.md:648-657), which is what ``oracle.max_marginals`` computes (fp64 C, pinned to brute force).
  Line 10 of Algorithm 5 is Eq. 21 / Theorem 4: x*_k = argmax_x psi~f_k psi~b_k,
  smallest index on ties.  SPEC's coherence diagnostic: the joint
  log-weight (Eq. 6) of the assembled path against the per-step optimum max_x log psi~f + log psi~b
  (= the MAP weight by Theorem 4), and the count of tied steps.
* ``viterbi_path_elements`` — Definition 4: elements a~_{i:j} = (A_{i:j}(x_i, x_j),
  X^_{i:j}(x_i, x_j)) combined by the operator v, base elements of Eq. 19, folded
  left to right (associativity, Lemma 2, makes the order immaterial for the values); by Corollary 1
   the total a~_{0:T+1} holds the MAP weight and the MAP path x*_{1:T}.  Log domain
  (max-plus is the log image of the products).  Ties: smallest x^_j at every combine.

Parity status: pinned (tests/test_oracle_pins.py: brute force on tie-free tiny inputs, a closed-form
incoherent tie case, the Algorithm 4 oracle on near-tie-free GE sequences).
"""
from __future__ import annotations

import numpy as np

from . import joint_weight, max_marginals

PATH_ELEMENT_MAX_T = 1024  # "the memory requirements to store the state sequences are high"


def viterbi_maxproduct(log_pi, log_A, log_lik, tie_tol: float = 0.0):
    """Algorithm 5.  Returns dict(path [T] int32 (Eq. 21), log_prob (per-step optimum at k = T, which by
    Theorem 4 is the MAP weight), path_weight (Eq. 6 joint log-weight of the assembled path),
    n_tied (#steps whose best and second-best max-marginal scores differ by <= tie_tol),
    coherent (path_weight attains log_prob to 1e-9 relative))."""
    ll = np.asarray(log_lik, np.float32)
    T, D = ll.shape
    score, gap = max_marginals(log_pi, log_A, ll)        # lines 1-8: log psi~f_k + log psi~b_k
    path = np.argmax(score, axis=1).astype(np.int32)      # line 10 / Eq. 21 (argmax: first maximum)
    log_prob = float(np.max(score[T - 1]))                # psi~b_T = 1 (Lemma 3 initial condition)
    w = joint_weight(log_pi, log_A, ll, path)
    n_tied = int(np.sum(gap <= tie_tol)) if D > 1 else 0
    coherent = bool(w >= log_prob - 1e-9 * max(1.0, abs(log_prob)))
    return dict(path=path, log_prob=log_prob, path_weight=w, n_tied=n_tied, coherent=coherent,
                score=score, gap=gap)


def viterbi_path_elements(log_pi, log_A, log_lik):
    """Definition 4 / Corollary 1 for T <= PATH_ELEMENT_MAX_T.  Returns dict(path [T] int32, log_prob)."""
    lp = np.asarray(log_pi, np.float32).astype(np.float64)
    la = np.asarray(log_A, np.float32).astype(np.float64)
    ll = np.asarray(log_lik, np.float32).astype(np.float64)
    T, D = ll.shape
    if T > PATH_ELEMENT_MAX_T:
        raise ValueError(f"T={T} exceeds the path-element cap {PATH_ELEMENT_MAX_T}")
    # a~_{0:1}: A_{0:1}(., x_1) = psi_1(x_1) (row-constant in the dummy x_0), X^ = empty  (Eq. 19)
    acc_A = np.tile(lp + ll[0], (D, 1))                   # [x_0, x_1]
    acc_X = np.zeros((D, D, 0), np.int64)                 # interior states x_1..x_{j-1}
    # a~_{k-1:k} (k = 2..T): A = log psi_{k-1,k}(x_{k-1}, x_k) = log A + log p(y_k | x_k); then the
    # terminal a~_{T:T+1} = (1, empty): psi = 1 for every pair (row of x_T, dummy x_{T+1})
    for t in range(1, T + 1):
        R = la + ll[t][None, :] if t < T else np.zeros((D, D))
        # a~_{i:k} = a~_{i:j} v a~_{j:k}: max over x_j of A_{i:j}(x_i, x_j) A_{j:k}(x_j, x_k)
        cand = acc_A[:, :, None] + R[None, :, :]          # [x_i, x_j, x_k]
        xh = np.argmax(cand, axis=1)                      # x^_j(x_i, x_k), smallest index on ties
        new_A = np.take_along_axis(cand, xh[:, None, :], axis=1)[:, 0, :]
        # X^_{i:k}(x_i, x_k) = (X^_{i:j}(x_i, x^_j), x^_j, X^_{j:k}(x^_j, x_k)); X^_{j:k} is empty here
        rows = np.arange(D)[:, None]
        new_X = np.concatenate([acc_X[rows, xh, :], xh[:, :, None]], axis=2)
        acc_A, acc_X = new_A, new_X
    # Corollary 1: a~_{0:T+1} = (psi_1(x*_1) prod psi(x*_{t-1}, x*_t), x*_{1:T}) for any dummy pair
    return dict(path=acc_X[0, 0, :].astype(np.int32), log_prob=float(acc_A[0, 0]))
