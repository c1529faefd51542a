"""GPU parity of variable-length batches and per-sequence models through the C ABI
(hmm_smooth_varlen / hmm_viterbi_varlen): every packed sequence is compared with the fp64 oracle run on
that sequence alone, with its own model (Eq. 5 potentials)."""
import numpy as np
import pytest
import torch

import oracle
import workloads as W
import paper_2102_05743_b200 as H
from parity import TAU, TOL_MARG, TOL_REL, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    H.lib()


def _batch(D, lengths, seed, per_seq, jitter=0.1):
    """Packed sequences: dense Dirichlet models + Gaussian emissions (config ③/④ recipe), jittered so the
    Viterbi paths are near-tie-free; per_seq draws one model per sequence."""
    rng_models = []
    lls = []
    for b, T in enumerate(lengths):
        wl = W.dense(D, int(T), seed=seed + b, model_seed=(7000 + seed + b) if per_seq else 424242 + D)
        ll = wl.log_lik + W.random_potentials(D, int(T), seed=99 + seed + b, sigma=jitter).log_lik
        rng_models.append((wl.log_pi, wl.log_A))
        lls.append(ll.astype(np.float32))
    off = np.zeros(len(lengths) + 1, np.int64)
    off[1:] = np.cumsum(lengths)
    return rng_models, lls, off


def _run(D, models, lls, off, per_seq, max_T=None):
    dev = torch.device("cuda")
    if per_seq:
        lp = torch.from_numpy(np.stack([m[0] for m in models])).to(dev)
        la = torch.from_numpy(np.stack([m[1] for m in models])).to(dev)
    else:
        lp = torch.from_numpy(models[0][0]).to(dev)
        la = torch.from_numpy(models[0][1]).to(dev)
    ll = torch.from_numpy(np.concatenate(lls)).to(dev)
    o = torch.from_numpy(off).to(dev)
    mt = max(len(x) for x in lls) if max_T is None else max_T
    f, s, lz, info = H.smooth_varlen(lp, la, ll, o, mt)
    path, lpr, vinfo = H.viterbi_varlen(lp, la, ll, o, mt)
    torch.cuda.synchronize()
    return [x.cpu().numpy() for x in (f, s, lz, info, path, lpr, vinfo)]


def _check(models, lls, off, res, per_seq):
    f, s, lz, info, path, lpr, vinfo = res
    for b, ll in enumerate(lls):
        lp, la = models[b] if per_seq else models[0]
        a, e = off[b], off[b + 1]
        o = oracle.smooth(lp, la, ll)
        assert int(info[b]) == 0 and int(vinfo[b]) == 0, (b, info[b], vinfo[b])
        assert float(np.abs(s[a:e] - o["smoothed"]).max()) <= TOL_MARG, b
        assert float(np.abs(f[a:e] - o["filtered"]).max()) <= TOL_MARG, b
        assert rel(float(lz[b]), o["log_z"]) <= TOL_REL, b
        v = oracle.viterbi(lp, la, ll)
        assert rel(float(lpr[b]), v["log_prob"]) <= TOL_REL, b
        _, gap = oracle.max_marginals(lp, la, ll)
        p = path[a:e]
        assert np.array_equal(p[gap >= TAU], v["path"][gap >= TAU]), b
        assert rel(oracle.joint_weight(lp, la, ll, p), v["log_prob"]) <= TOL_REL, b


@pytest.mark.parametrize("D", [1, 2, 3, 4, 7, 8, 12, 16, 33])
@pytest.mark.parametrize("per_seq", [False, True])
def test_varlen_vs_oracle(D, per_seq):
    rng = np.random.default_rng(D * 10 + per_seq)
    lengths = rng.integers(1, 2500, size=23)
    lengths[:3] = [1, 2, 2499]
    models, lls, off = _batch(D, lengths, seed=D, per_seq=per_seq)
    res = _run(D, models, lls, off, per_seq)
    _check(models, lls, off, res, per_seq)


def test_varlen_config4_like():
    """Config ④'s shape with ragged lengths: B=1024, D=16, T_b ~ U[256, 4096], per-sequence models."""
    rng = np.random.default_rng(4)
    lengths = rng.integers(256, 4097, size=1024)
    models, lls, off = _batch(16, lengths, seed=1000, per_seq=True)
    res = _run(16, models, lls, off, True, max_T=4096)
    sel = list(range(0, 1024, 37)) + [1023]
    f, s, lz, info, path, lpr, vinfo = res
    assert (info == 0).all() and (vinfo == 0).all()
    for b in sel:
        lp, la = models[b]
        a, e = off[b], off[b + 1]
        o = oracle.smooth(lp, la, lls[b])
        assert float(np.abs(s[a:e] - o["smoothed"]).max()) <= TOL_MARG
        assert rel(float(lz[b]), o["log_z"]) <= TOL_REL
        v = oracle.viterbi(lp, la, lls[b])
        assert rel(float(lpr[b]), v["log_prob"]) <= TOL_REL
        assert rel(oracle.joint_weight(lp, la, lls[b], path[a:e]), v["log_prob"]) <= TOL_REL


@pytest.mark.parametrize("D", [4, 16])
def test_varlen_equal_lengths_match_batched(D):
    """All lengths equal: the varlen call returns what the batched call returns (same arithmetic to
    within the tolerances; D <= 8 batched plans may split a sequence over several CTAs)."""
    B, T = 9, 1500
    wl = W.dense_batch(B, D, T)
    dev = torch.device("cuda")
    lp, la = torch.from_numpy(wl.log_pi).to(dev), torch.from_numpy(wl.log_A).to(dev)
    ll3 = torch.from_numpy(wl.log_lik).to(dev)
    off = torch.arange(0, (B + 1) * T, T, dtype=torch.int64, device=dev)
    f1, s1, lz1, i1 = H.smooth(lp, la, ll3)
    f2, s2, lz2, i2 = H.smooth_varlen(lp, la, ll3.reshape(B * T, D), off, T)
    p1, q1, _ = H.viterbi(lp, la, ll3)
    p2, q2, _ = H.viterbi_varlen(lp, la, ll3.reshape(B * T, D), off, T)
    torch.cuda.synchronize()
    assert float((s1.reshape(B * T, D) - s2).abs().max()) <= 2 * TOL_MARG
    assert float(((lz1 - lz2).abs() / lz1.abs()).max()) <= 2 * TOL_REL
    assert float(((q1 - q2).abs() / q1.abs()).max()) <= 2 * TOL_REL


@pytest.mark.parametrize("D", [4, 16])
def test_varlen_bad_lengths(D):
    lengths = [5, 7, 9]
    models, lls, off = _batch(D, lengths, seed=3, per_seq=False)
    dev = torch.device("cuda")
    lp, la = (torch.from_numpy(x).to(dev) for x in models[0])
    ll = torch.from_numpy(np.concatenate(lls)).to(dev)
    bad = torch.tensor([0, 5, 5, 21], dtype=torch.int64, device=dev)  # sequence 1 empty, sequence 2 > max_T
    f, s, lz, info = H.smooth_varlen(lp, la, ll, bad, 10)
    path, lpr, vinfo = H.viterbi_varlen(lp, la, ll, bad, 10)
    torch.cuda.synchronize()
    assert info.tolist() == [0, H.HMM_INFO_BAD_LENGTH, H.HMM_INFO_BAD_LENGTH]
    assert vinfo.tolist() == [0, H.HMM_INFO_BAD_LENGTH, H.HMM_INFO_BAD_LENGTH]
    o = oracle.smooth(*models[0], lls[0])
    assert float(np.abs(s[:5].cpu().numpy() - o["smoothed"]).max()) <= TOL_MARG


def test_varlen_impossible_step_per_sequence():
    lengths = [300, 400, 500]
    models, lls, off = _batch(4, lengths, seed=5, per_seq=True)
    lls[1][123, :] = -np.inf
    res = _run(4, models, lls, off, True)
    f, s, lz, info, path, lpr, vinfo = res
    assert info.tolist() == [0, 124, 0] and vinfo.tolist() == [0, 124, 0]


@pytest.mark.parametrize("D", [2, 4, 8])
def test_varlen_long_sequences_chunked(D):
    """D <= 8 runs one CTA per sequence: a long member (T = 400 003) takes the chunked resident plan
    (many chunks per CTA, chunk roots and backpointers in the workspace) next to short members."""
    lengths = [400_003, 17, 65_537, 1]
    models, lls, off = _batch(D, lengths, seed=40 + D, per_seq=True)
    res = _run(D, models, lls, off, True)
    _check(models, lls, off, res, True)


@pytest.mark.parametrize("D", [9, 12, 16, 20, 32])
def test_varlen_batch_plan_chunk_edges(D):
    """The bidirectional batch plan forced on ragged lengths at its chunk edges (16-step smoother chunks,
    32-step Viterbi chunks, mid = ceil(chunks / 2)): lengths 1, 15..17, 31..33, 47..49, 63..65, 95..97 and
    a long one, an odd batch (an idle lane group at D <= 16), per-sequence models; every sequence vs the
    oracle."""
    lengths = [1, 15, 16, 17, 31, 32, 33, 47, 48, 49, 63, 64, 65, 95, 96, 97, 1000]
    models, lls, off = _batch(D, lengths, seed=300 + D, per_seq=True)
    H.force_path(4)
    try:
        res = _run(D, models, lls, off, True)
    finally:
        H.force_path(0)
    _check(models, lls, off, res, True)
