"""GPU parity of the paper-faithful Viterbi variants through the C ABI:

* hmm_viterbi_maxproduct — Algorithm 5: Eq. 21 per-step argmax of the forward and
  reversed max-product scans, with SPEC's coherence diagnostic;
* hmm_viterbi_path_elements — the Definition 4 path-element reduction (Corollary 1).

Compared with ``oracle.variants`` (fp64, pinned to brute force) on tie-free inputs (bit-exact paths),
at gap >= TAU elsewhere, and on raw GE observations, whose exact ties must be flagged.
"""
import numpy as np
import pytest
import torch

import oracle
from oracle import variants as OV
import workloads as W
import paper_2102_05743_b200 as H
from parity import TAU, TOL_REL, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    H.lib()


def _dev(wl):
    d = torch.device("cuda")
    return tuple(torch.from_numpy(np.ascontiguousarray(x)).to(d) for x in (wl.log_pi, wl.log_A, wl.log_lik))


def _a5(wl, tie_tol=0.0):
    lp, la, ll = _dev(wl)
    out = H.viterbi_maxproduct(lp, la, ll, tie_tol=tie_tol)
    torch.cuda.synchronize()
    return [x.cpu().numpy() for x in out]


def _pe(wl):
    lp, la, ll = _dev(wl)
    out = H.viterbi_path_elements(lp, la, ll)
    torch.cuda.synchronize()
    return [x.cpu().numpy() for x in out]


def _check_a5(wl, path, lp, pw, nt, info, b=None, expect_coherent=None):
    ll = wl.log_lik if b is None else wl.log_lik[b]
    i = 0 if b is None else b
    p = path if b is None else path[b]
    o = OV.viterbi_maxproduct(wl.log_pi, wl.log_A, ll)
    assert rel(float(lp[i]), o["log_prob"]) <= TOL_REL
    # the device's fp64 path weight is Eq. 6 of the returned path: equal to the oracle's evaluation
    jw = oracle.joint_weight(wl.log_pi, wl.log_A, ll, p)
    assert abs(float(pw[i]) - jw) <= 1e-9 * max(1.0, abs(jw))
    safe = o["gap"] >= TAU
    mism = np.nonzero((p != o["path"]) & safe)[0]
    assert mism.size == 0, f"{mism.size} Eq. 21 mismatches at gap >= TAU, first {mism[:5]}"
    coherent = jw >= o["log_prob"] - 1e-6 * max(1.0, abs(o["log_prob"]))
    assert int(info[i]) == (0 if coherent else H.HMM_INFO_AMBIGUOUS)
    if expect_coherent is not None:
        assert coherent == expect_coherent
    return o


@pytest.mark.parametrize("D", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("T", [1, 2, 17, 4097, 100_003])
def test_alg5_tie_free_exact(D, T):
    """Jittered random potentials: no near-ties, so Eq. 21 gives the MAP path bit for bit (Theorem 4)."""
    wl = W.random_potentials(D, T, seed=11 * D + T % 97)
    path, lp, pw, nt, info = _a5(wl)
    o = _check_a5(wl, path, lp, pw, nt, info)
    if o["gap"].min() >= TAU:
        np.testing.assert_array_equal(path, o["path"])
        v = oracle.viterbi(wl.log_pi, wl.log_A, wl.log_lik)
        np.testing.assert_array_equal(path, v["path"])  # = Algorithm 4's MAP path
        assert int(info[0]) == 0


@pytest.mark.parametrize("T", [1000, 1_000_000])
def test_alg5_ge_jittered(T):
    wl = W.ge(T, seed=1, jitter=0.1)
    path, lp, pw, nt, info = _a5(wl)
    _check_a5(wl, path, lp, pw, nt, info)


def test_alg5_raw_ge_flags_ties():
    """Raw GE observations: exact max-marginal ties.  n_tied counts the exactly tied
    steps (fp32 on the device); the diagnostic reports HMM_INFO_AMBIGUOUS iff the assembly falls below
    the MAP weight, in agreement with the oracle's evaluation of the returned path."""
    wl = W.ge(10_000, seed=0)
    path, lp, pw, nt, info = _a5(wl)
    o = _check_a5(wl, path, lp, pw, nt, info)
    assert int(nt[0]) > 0 and o["n_tied"] > 0
    # the production Viterbi on the same input returns a MAP path (backpointers are exact under ties)
    lpd, lad, lld = _dev(wl)
    vp, vlp, vinfo = H.viterbi(lpd, lad, lld)
    assert abs(oracle.joint_weight(wl.log_pi, wl.log_A, wl.log_lik, vp.cpu().numpy()) - o["log_prob"]) <= \
        1e-6 * abs(o["log_prob"])


def test_alg5_incoherent_closed_form():
    """Alternating two-state chain (oracle pin test_alg5_incoherent_under_ties_closed_form): every step
    is tied, Eq. 21 assembles the all-zero path, whose weight is below the MAP: info = AMBIGUOUS."""
    eps, T = 0.1, 4099
    lp = np.log(np.array([0.5, 0.5])).astype(np.float32)
    la = np.log(np.array([[eps, 1 - eps], [1 - eps, eps]])).astype(np.float32)
    ll = np.zeros((T, 2), np.float32)
    wl = W.Workload(lp, la, ll, None, "alternating")
    path, lpv, pw, nt, info = _a5(wl)
    np.testing.assert_array_equal(path, np.zeros(T, np.int32))
    assert int(nt[0]) == T and int(info[0]) == H.HMM_INFO_AMBIGUOUS
    map_w = float(np.float64(lp[0]) + (T - 1) * np.float64(la[0, 1]))
    assert rel(float(lpv[0]), map_w) <= TOL_REL


def test_alg5_batched_and_info():
    wl = W.random_potentials(4, 3001, seed=5, B=5)
    wl.log_lik[2, 1234, :] = -np.inf      # impossible step in sequence 2
    wl.log_lik[4, 17, 1] = np.nan         # bad input in sequence 4
    path, lp, pw, nt, info = _a5(wl)
    assert int(info[2]) == 1235 and int(info[4]) == -1
    for b in (0, 1, 3):
        _check_a5(wl, path, lp, pw, nt, info, b=b)


def test_alg5_deterministic():
    wl = W.ge(300_001, seed=2)
    a = _a5(wl)
    b = _a5(wl)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("D", [1, 2, 3, 4, 6, 8])
@pytest.mark.parametrize("T", [1, 2, 3, 64, 1000, 1024])
def test_path_elements_vs_oracle(D, T):
    wl = W.random_potentials(D, T, seed=3 * D + T)
    path, lp, info = _pe(wl)
    o = OV.viterbi_path_elements(wl.log_pi, wl.log_A, wl.log_lik)
    assert int(info[0]) == 0
    assert rel(float(lp[0]), o["log_prob"]) <= TOL_REL
    _, gap = oracle.max_marginals(wl.log_pi, wl.log_A, wl.log_lik)
    safe = gap >= TAU
    assert np.array_equal(path[safe], o["path"][safe])
    jw = oracle.joint_weight(wl.log_pi, wl.log_A, wl.log_lik, path)
    assert rel(jw, o["log_prob"]) <= TOL_REL


def test_path_elements_ge_batched_ties():
    """Raw GE (ties): the reduction still returns a MAP path (Corollary 1) for every sequence."""
    B, T = 6, 1024
    lls = np.stack([W.ge(T, seed=s).log_lik for s in range(B)])
    g = W.ge(T, seed=0)
    wl = W.Workload(g.log_pi, g.log_A, lls, None, "ge_batch")
    path, lp, info = _pe(wl)
    for b in range(B):
        v = oracle.viterbi(wl.log_pi, wl.log_A, lls[b])
        assert int(info[b]) == 0
        assert rel(float(lp[b]), v["log_prob"]) <= TOL_REL
        assert rel(oracle.joint_weight(wl.log_pi, wl.log_A, lls[b], path[b]), v["log_prob"]) <= TOL_REL


def test_path_elements_cap_and_no_path():
    wl = W.ge(H.HMM_PATHELEM_MAX_T + 1, seed=0)
    with pytest.raises(H.HmmError):
        _pe(wl)
    wl = W.ge(50, seed=0)
    wl.log_lik[20, :] = -np.inf
    path, lp, info = _pe(wl)
    assert int(info[0]) == H.HMM_INFO_NO_PATH
