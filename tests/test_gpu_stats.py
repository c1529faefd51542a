"""GPU parity of the Baum-Welch E-step statistics fused into
the lane-streaming smoother's backward sweep (hmm_smooth_stats): xi_sum and gamma_sum vs the fp64
oracle (oracle.smooth_stats, itself pinned to enumeration).  Bar: every entry within 1e-5 relative
(absolute for entries below 1) -- the marginal bar of BASELINE.json applied to sums of marginals --
plus the exact invariant sum(xi) = T - 1 to 1e-6 relative."""
import numpy as np
import pytest
import torch

import oracle
import workloads as W
import paper_2102_05743_b200 as H
from parity import TOL_MARG, TOL_REL, rel, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    H.lib()


def _check(wl, res):
    f, s, lz, xi, g, info = res
    torch.cuda.synchronize()
    o = oracle.smooth_stats(wl.log_pi, wl.log_A, wl.log_lik)
    assert int(info[0]) == 0 and o["info"] == 0
    xi, g = xi.cpu().numpy(), g.cpu().numpy()
    assert (np.abs(xi - o["xi_sum"]) <= 1e-5 * np.maximum(np.abs(o["xi_sum"]), 1.0)).all()
    assert (np.abs(g - o["gamma_sum"]) <= 1e-5 * np.maximum(np.abs(o["gamma_sum"]), 1.0)).all()
    T = wl.log_lik.shape[0]
    assert abs(xi.sum() - (T - 1)) <= 1e-6 * max(T, 1) + 1e-6
    assert rel(float(lz[0]), o["log_z"]) <= TOL_REL
    if s is not None:
        m = oracle.smooth(wl.log_pi, wl.log_A, wl.log_lik)
        assert float(np.abs(s.cpu().numpy() - m["smoothed"]).max()) <= TOL_MARG
        assert float(np.abs(f.cpu().numpy() - m["filtered"]).max()) <= TOL_MARG


@pytest.mark.parametrize("D", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("T", [1, 2, 17, 20_011])
def test_stats_every_D(D, T):
    wl = W.ge(T, 3) if D == 4 else W.dense(D, T, 3)
    _check(wl, H.smooth_stats(*to_dev(wl)))


@pytest.mark.parametrize("D,T", [(4, 2_000_003), (8, 300_001), (2, 1_000_000)])
def test_stats_long(D, T):
    wl = W.ge(T, 9) if D == 4 else W.dense(D, T, 9)
    _check(wl, H.smooth_stats(*to_dev(wl)))


def test_stats_only_and_deterministic():
    wl = W.ge(1_000_003, 4)
    a = H.smooth_stats(*to_dev(wl), want_marginals=False)
    b = H.smooth_stats(*to_dev(wl), want_marginals=False)
    assert a[0] is None and a[1] is None
    _check(wl, a)
    for x, y in zip(a[2:], b[2:]):
        assert torch.equal(x, y)


def test_stats_unnormalised_potentials():
    wl = W.random_potentials(4, 50_000, seed=8)
    _check(wl, H.smooth_stats(*to_dev(wl)))


def test_stats_info_impossible_step():
    wl = W.ge(300_000, 6)
    wl.log_lik[123_456, :] = -np.inf
    assert int(H.smooth_stats(*to_dev(wl))[5][0]) == 123_457


def test_stats_mstep_transition_estimate():
    """One EM step on a long GE sequence: the re-estimated transition matrix A' = xi / rowsum(xi)
    matches the oracle's to 1e-6 (what a Baum-Welch user consumes)."""
    wl = W.ge(3_000_000, 12)
    _, _, _, xi, _, _ = H.smooth_stats(*to_dev(wl), want_marginals=False)
    xi = xi.cpu().numpy()
    o = oracle.smooth_stats(wl.log_pi, wl.log_A, wl.log_lik)["xi_sum"]
    A1 = xi / xi.sum(1, keepdims=True); A0 = o / o.sum(1, keepdims=True)
    assert float(np.abs(A1 - A0).max()) <= 1e-6
