"""GPU parity of the batch-parallel plan for 9 <= D <= 32 (hmm_batchseq.cu): one lane
group per sequence runs Algorithm 1's forward/backward passes and Algorithm 4's max-product pass with
backpointers (the sequence is one block-wise element).
Forced with hmm_debug_force_path(4) on small batches, compared with the fp64 oracle per sequence and
with the block-scan plan (force 5) on the same inputs."""
import numpy as np
import pytest
import torch

import oracle
import workloads as W
import paper_2102_05743_b200 as H
from parity import TAU, TOL_MARG, TOL_REL, rel, check_smooth, check_viterbi

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    H.lib()


def _run(wl, force):
    d = torch.device("cuda")
    lp, la, ll = (torch.from_numpy(np.ascontiguousarray(x)).to(d) for x in (wl.log_pi, wl.log_A, wl.log_lik))
    H.force_path(force)
    try:
        f, s, lz, info = H.smooth(lp, la, ll)
        p, q, vinfo = H.viterbi(lp, la, ll)
        torch.cuda.synchronize()
    finally:
        H.force_path(0)
    return [x.cpu().numpy() for x in (f, s, lz, info)], [x.cpu().numpy() for x in (p, q, vinfo)]


@pytest.mark.parametrize("force", [4, 6], ids=["bidir", "one_warp"])
@pytest.mark.parametrize("D", [9, 12, 16, 17, 25, 32])
@pytest.mark.parametrize("T", [1, 2, 7, 31, 32, 33, 64, 65, 1000, 4099])
def test_batchseq_vs_oracle(D, T, force):
    """force 4: the bidirectional plan (two warps per sequence, forward and backward recursions from both
    ends, meeting at mid = ceil(chunks / 2); T around the 32-step chunk covers mid = T and a one-row
    second half); force 6: the one-warp plan."""
    wl = W.dense_batch(5, D, T, model_seed=77 + D, seed0=31 * T)
    wl.log_lik = wl.log_lik + W.random_potentials(D, T, seed=D, B=5, sigma=0.1).log_lik  # near-tie-free
    s, v = _run(wl, force)
    for b in range(5):
        check_smooth(wl, *s, b=b)
        check_viterbi(wl, *v, b=b)


@pytest.mark.parametrize("D", [16, 32])
def test_batchseq_unnormalised_and_scan_agree(D):
    wl = W.random_potentials(D, 3000, seed=4, B=3)
    s4, v4 = _run(wl, 4)
    s5, v5 = _run(wl, 5)
    for b in range(3):
        check_smooth(wl, *s4, b=b)
        check_viterbi(wl, *v4, b=b)
    assert float(np.abs(s4[1] - s5[1]).max()) <= 2 * TOL_MARG
    assert float(np.max(np.abs(s4[2] - s5[2]) / np.abs(s5[2]))) <= 2 * TOL_REL


def test_batchseq_info_codes():
    wl = W.random_potentials(16, 2000, seed=9, B=4)
    wl.log_lik[1, 777, :] = -np.inf
    wl.log_lik[2, 5, 3] = np.nan
    s, v = _run(wl, 4)
    assert s[3].tolist() == [0, 778, -1, 0]
    assert v[2].tolist() == [0, 778, -1, 0]


def test_batchseq_is_the_auto_plan_for_config4_shape():
    """B = 1024, D = 16: the planner takes the batch-parallel plan (config ④) — checked by comparing the
    automatic result bitwise with the forced plan."""
    wl = W.dense_batch(1024, 16, 256)
    a, av = _run(wl, 0)
    f, fv = _run(wl, 4)
    np.testing.assert_array_equal(a[1], f[1])
    np.testing.assert_array_equal(av[0], fv[0])
    for b in (0, 100, 1023):
        check_smooth(wl, *a, b=b)


def test_batchseq_varlen_per_sequence_models():
    rng = np.random.default_rng(2)
    B, D = 200, 32
    lengths = rng.integers(1, 1500, size=B)
    models, lls = [], []
    for b in range(B):
        w = W.dense(D, int(lengths[b]), seed=b, model_seed=5000 + b)
        models.append((w.log_pi, w.log_A)); lls.append(w.log_lik)
    off = np.zeros(B + 1, np.int64); off[1:] = np.cumsum(lengths)
    d = torch.device("cuda")
    lp = torch.from_numpy(np.stack([m[0] for m in models])).to(d)
    la = torch.from_numpy(np.stack([m[1] for m in models])).to(d)
    ll = torch.from_numpy(np.concatenate(lls)).to(d)
    o = torch.from_numpy(off).to(d)
    f, s, lz, info = H.smooth_varlen(lp, la, ll, o, int(lengths.max()))   # D = 32, B >= 160: batch-parallel
    p, q, vinfo = H.viterbi_varlen(lp, la, ll, o, int(lengths.max()))
    torch.cuda.synchronize()
    s, lz, p, q = s.cpu().numpy(), lz.cpu().numpy(), p.cpu().numpy(), q.cpu().numpy()
    assert (info.cpu().numpy() == 0).all() and (vinfo.cpu().numpy() == 0).all()
    for b in range(0, B, 13):
        a, e = off[b], off[b + 1]
        or_ = oracle.smooth(*models[b], lls[b])
        assert float(np.abs(s[a:e] - or_["smoothed"]).max()) <= TOL_MARG
        assert rel(float(lz[b]), or_["log_z"]) <= TOL_REL
        v = oracle.viterbi(*models[b], lls[b])
        assert rel(float(q[b]), v["log_prob"]) <= TOL_REL
        assert rel(oracle.joint_weight(*models[b], lls[b], p[a:e]), v["log_prob"]) <= TOL_REL


@pytest.mark.parametrize("D", [16, 32])
def test_batchseq_bidir_equals_one_warp(D):
    """Both batch-parallel variants on the same unnormalised inputs: filtered, smoothed and log Z within
    rounding (the dot products are summed in a different order), the MAP value within rounding of its
    offsets and the path equal (no ties in random potentials)."""
    wl = W.random_potentials(D, 2500, seed=9, B=6)
    s4, v4 = _run(wl, 4)
    s6, v6 = _run(wl, 6)
    assert float(np.abs(s4[0] - s6[0]).max()) <= TOL_MARG
    assert float(np.max(np.abs(s4[2] - s6[2]) / np.abs(s6[2]))) <= TOL_REL
    assert float(np.abs(s4[1] - s6[1]).max()) <= TOL_MARG
    assert np.array_equal(v4[0], v6[0])
    assert float(np.max(np.abs(v4[1] - v6[1]) / np.abs(v6[1]))) <= TOL_REL
    assert np.array_equal(s4[3], s6[3]) and np.array_equal(v4[2], v6[2])


def test_batchseq_bidir_impossible_second_half():
    """An impossible step in the backward warp's half: the meet sees -inf, the forward warp runs on to
    locate it (info = t + 1) exactly as the one-warp plan."""
    wl = W.dense_batch(3, 16, 700, model_seed=5, seed0=3)
    wl.log_lik = np.ascontiguousarray(wl.log_lik.copy())
    wl.log_lik[1, 600, :] = -np.inf
    s4, v4 = _run(wl, 4)
    s6, v6 = _run(wl, 6)
    assert s4[3][1] == 601 and v4[2][1] == 601
    assert np.array_equal(s4[3], s6[3]) and np.array_equal(v4[2], v6[2])
    for b in (0, 2):
        check_smooth(wl, *s4, b=b)
        check_viterbi(wl, *v4, b=b)
