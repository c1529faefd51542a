"""GPU parity of the lane-streaming kernel (hmm_stream.cu) and of the path selection around it.

The library picks the streaming decomposition for long single sequences and for every split-phase
call; `H.force_path` (hmm_debug_force_path) pins a decomposition so that each one is compared with
the fp64 oracle at sizes the oracle finishes in seconds, across every D, ragged T and multi-slice
lanes.  The last tests run BASELINE config 5 at full size on one GPU (GE D=4, T=1e8, the launch
configuration bench.py times) and check sampled outputs against oracle.smooth_sampled, log Z and
log_prob against the oracle, and properties that hold at any size.
"""
import numpy as np
import pytest
import torch

import oracle
import workloads as W
import paper_2102_05743_b200 as H
from parity import TAU, TOL_MARG, TOL_REL, check_smooth, check_viterbi, gpu_smooth, gpu_viterbi, record, rel, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    H.lib()
    yield
    H.force_path(0)


@pytest.fixture
def stream():
    H.force_path(1)
    yield
    H.force_path(0)


def _wl(D, T, seed=3, jitter=0.0):
    return W.ge(T, seed, jitter=jitter) if D == 4 else W.dense(D, T, seed)


# ---------------------------------------------------------------- forced streaming path
@pytest.mark.parametrize("D", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("T", [1, 7, 4099, 20_011])
def test_stream_every_D_smoother(stream, D, T):
    wl = _wl(D, T)
    assert H.plan(0, D, T)["fused"] == 2
    check_smooth(wl, *gpu_smooth(wl))


@pytest.mark.parametrize("D", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("T", [1, 7, 4099, 20_011])
def test_stream_every_D_viterbi(stream, D, T):
    wl = _wl(D, T, jitter=0.1)
    check_viterbi(wl, *gpu_viterbi(wl))


@pytest.mark.parametrize("D,T", [(4, 2_000_003), (1, 3_000_001), (2, 1_500_000), (3, 1_000_001), (8, 600_001)])
def test_stream_multislice_lanes(stream, D, T):
    """Several slices per lane (K > 1), ragged last lane, and (T*D % 4 != 0) partial 16-B chunks."""
    pl = H.plan(0, D, T)
    assert pl["K"] > 1
    wl = _wl(D, T, seed=11)
    check_smooth(wl, *gpu_smooth(wl))
    wj = _wl(D, T, seed=12, jitter=0.1)
    check_viterbi(wj, *gpu_viterbi(wj))


def test_stream_planted_exact(stream):
    for D in (2, 5, 8):
        wp = W.planted(D, 500_000, seed=D)
        path, lp, info = gpu_viterbi(wp)
        assert int(info[0]) == 0 and np.array_equal(path, wp.states)


@pytest.mark.parametrize("T,t_bad", [(3_000_000, 2_500_001), (3_000_000, 0), (3_000_000, 2_999_999)])
def test_stream_info_impossible_evidence(stream, T, t_bad):
    wl = W.ge(T, seed=6)
    wl.log_lik[t_bad, :] = -np.inf
    _, _, _, info = gpu_smooth(wl)
    assert int(info[0]) == t_bad + 1
    _, _, vinfo = gpu_viterbi(wl)
    assert int(vinfo[0]) == t_bad + 1


def test_stream_info_nan_inf(stream):
    wl = W.ge(3_000_000, seed=7)
    wl.log_lik[1_654_321, 2] = np.nan
    assert int(gpu_smooth(wl)[3][0]) == -1
    assert int(gpu_viterbi(wl)[2][0]) == -1
    wl = W.ge(3_000_000, seed=7)
    wl.log_lik[3, 1] = np.inf
    assert int(gpu_smooth(wl)[3][0]) == -1


def test_stream_deterministic_and_workspace_left_zeroed(stream):
    wl = W.ge(3_000_000, seed=8)
    a = gpu_smooth(wl); b = gpu_smooth(wl)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    p1 = gpu_viterbi(wl); p2 = gpu_viterbi(wl)
    for x, y in zip(p1, p2):
        assert np.array_equal(x, y)
    for op in (H.HMM_OP_SMOOTH, H.HMM_OP_VITERBI):
        ws = H.workspace(op, 4, 3_000_000, 1)
        words = ws[:64].view(torch.int32).cpu().numpy()
        assert (words[:10] == 0).all()


def test_stream_filtered_null(stream):
    wl = W.ge(1_000_003, seed=5)
    f, s, lz, info = gpu_smooth(wl, want_filtered=False)
    assert f is None
    o = oracle.smooth(wl.log_pi, wl.log_A, wl.log_lik)
    assert float(np.abs(s - o["smoothed"]).max()) <= TOL_MARG
    assert rel(lz[0], o["log_z"]) <= TOL_REL


# ---------------------------------------------------------------- the other decompositions, same inputs
@pytest.mark.parametrize("T", [2_000_003, 5_000_000])
def test_forced_chunked_path_long_T(T):
    """The resident/chunked two-pass plan stays correct when selected for long sequences."""
    H.force_path(2)
    try:
        assert H.plan(0, 4, T)["fused"] in (0, 1)
        wl = W.ge(T, seed=3)
        check_smooth(wl, *gpu_smooth(wl))
        wj = W.ge(T, seed=4, jitter=0.1)
        check_viterbi(wj, *gpu_viterbi(wj))
    finally:
        H.force_path(0)


def test_unaligned_buffers_fall_back(stream):
    """A log_lik view that is not 16-B aligned cannot take the streaming kernel's coalesced copies:
    even with the streaming path requested the library falls back to the chunked plan, and the
    results are unchanged."""
    D, T = 1, 3_000_001
    wl = W.dense(D, T + 1, seed=2)
    dev = torch.device("cuda")
    ll_all = torch.from_numpy(wl.log_lik).to(dev)
    ll = ll_all[1:]  # 4-B offset
    assert ll.data_ptr() % 16 != 0
    lp, la = torch.from_numpy(wl.log_pi).to(dev), torch.from_numpy(wl.log_A).to(dev)
    f, s, lz, info = H.smooth(lp, la, ll)
    o = oracle.smooth(wl.log_pi, wl.log_A, wl.log_lik[1:])
    assert int(info[0]) == 0
    assert float(np.abs(s.cpu().numpy() - o["smoothed"]).max()) <= TOL_MARG
    assert rel(float(lz[0]), o["log_z"]) <= TOL_REL


def test_paths_agree_on_same_input():
    """Fused, chunked and streaming decompositions on the same input agree within the tolerances."""
    wl = W.ge(1_000_000, seed=21)
    res = {}
    for path in (0, 1, 2):
        H.force_path(path)
        res[path] = gpu_smooth(wl)
    H.force_path(0)
    for path in (1, 2):
        assert float(np.abs(res[path][1] - res[0][1]).max()) <= 2 * TOL_MARG
        assert rel(res[path][2][0], res[0][2][0]) <= TOL_REL


# ---------------------------------------------------------------- BASELINE config 5 at full size, 1 GPU
T_FULL = 100_000_000


@pytest.fixture(scope="module")
def full_ge():
    return W.ge(T_FULL, 5)


def _lane_boundary_steps(T, D=4):
    """Every step where the lane-streaming decomposition changes hands: first and last step of every
    lane (CTA boundaries are lane boundaries), plus every slice boundary of a few lanes."""
    pl = H.plan(0, D, T)
    assert pl["fused"] == 2
    n, S, lanes = pl["R"], pl["S"], pl["G"] * pl["NT"]
    starts = np.arange(lanes, dtype=np.int64) * n
    starts = starts[starts < T]
    ts = [starts, starts - 1, np.minimum(starts + n - 1, T - 1)]
    for g in (0, 1, len(starts) // 2, len(starts) - 1):
        ks = starts[g] + np.arange(0, n, S, dtype=np.int64)
        ts += [ks, ks - 1]
    ts = np.concatenate(ts)
    return np.unique(ts[(ts >= 0) & (ts < T)]), pl


def test_config5_full_size_smoother(full_ge):
    """Config 5 at full size: every lane start / end and CTA boundary (where the lane chains and the
    carries meet) plus random steps against the exact fp64 recursions (Alg. 1 + Eq. 14)."""
    wl = full_ge
    dev = torch.device("cuda")
    lp, la, ll = to_dev(wl)
    f, s, lz, info = H.smooth(lp, la, ll)
    torch.cuda.synchronize()
    assert int(info[0]) == 0
    # properties at every step: rows are distributions
    for x in (f, s):
        assert float((x.sum(1) - 1).abs().max()) <= 1e-5
        assert float(x.min()) >= 0.0
    rng = np.random.default_rng(0)
    tb, pl = _lane_boundary_steps(T_FULL)
    ts = np.unique(np.r_[tb, 0, 1, T_FULL - 1, rng.integers(0, T_FULL, 20000)])
    o = oracle.smooth_sampled(wl.log_pi, wl.log_A, wl.log_lik, ts)
    tt = torch.from_numpy(ts).to(dev)
    ef = np.abs(f[tt].cpu().numpy() - o["filtered"]).max(1)
    es = np.abs(s[tt].cpu().numpy() - o["smoothed"]).max(1)
    r = rel(float(lz[0]), o["log_z"])
    record("config5_smoother_T1e8", samples=int(ts.size), lane_boundaries=int(tb.size), lane_steps=pl["R"],
           lanes=pl["G"] * pl["NT"], max_err_filtered=ef.max(), max_err_smoothed=es.max(),
           worst_step_smoothed=int(ts[es.argmax()]), mean_err_smoothed=es.mean(), log_z_rel=r)
    assert float(ef.max()) <= TOL_MARG
    assert float(es.max()) <= TOL_MARG
    assert r <= TOL_REL


def test_config5_full_size_viterbi():
    """Config 5 at full size (near-tie-free GE copy): the path is bit-exact at EVERY one of the 1e8 steps
    whose oracle max-marginal gap is >= TAU (O(T)-memory gap, Lemma 3), and where it differs the GPU path
    loses at most 1e-3 nats of joint log-probability against the MAP (Eq. 6, compared term by term)."""
    wl = W.ge(T_FULL, 5, jitter=0.1)
    lp, la, ll = to_dev(wl)
    path, lpr, info = H.viterbi(lp, la, ll)
    torch.cuda.synchronize()
    assert int(info[0]) == 0
    v = oracle.viterbi(wl.log_pi, wl.log_A, wl.log_lik)
    r = rel(float(lpr[0]), v["log_prob"])
    gp = path.cpu().numpy()
    del path, ll
    gap = oracle.max_marginal_gap(wl.log_pi, wl.log_A, wl.log_lik)
    safe = gap >= TAU
    diff = gp != v["path"]
    mism = int((diff & safe).sum())
    dw = oracle.joint_weight_diff(wl.log_pi, wl.log_A, wl.log_lik, gp, v["path"])
    record("config5_viterbi_T1e8", masked_positions=int((~safe).sum()), differing_positions=int(diff.sum()),
           mismatches_at_gap_ge_tau=mism, joint_weight_gpu_minus_map=dw, log_prob_rel=r,
           log_prob_abs=abs(float(lpr[0]) - v["log_prob"]))
    assert mism == 0, f"{mism} mismatches at near-tie-free positions"
    assert -1e-3 <= dw <= 1e-6, f"GPU path joint log-prob - MAP = {dw} nats"
    assert r <= TOL_REL


def test_config5_full_size_planted_exact():
    wp = W.planted(4, T_FULL, seed=4)
    lp, la, ll = to_dev(wp)
    path, lpr, info = H.viterbi(lp, la, ll)
    assert int(info[0]) == 0
    assert torch.equal(path.cpu(), torch.from_numpy(wp.states))
