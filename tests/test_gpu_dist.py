"""Split-phase (multi-GPU) kernels emulated on one GPU: W ranks' reduce / finish phases run in
sequence through the C ABI with per-rank workspaces, the all-gathers are host-side concatenations in
rank order (what NCCL's all_gather_into_tensor produces).  Results must match the fp64 oracle on the
unpartitioned sequence and the single-call path (rank-count invariance)."""
import numpy as np
import pytest
import torch

import oracle
import workloads as W
from parity import TAU, TOL_MARG, TOL_REL, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _slices(T, world):
    from paper_2102_05743_b200.dist import partition
    return [partition(T, world, r) for r in range(world)]


def emulate_smooth(wl, world):
    from paper_2102_05743_b200.dist import LibBackend
    dev = torch.device("cuda")
    lp, la = torch.from_numpy(wl.log_pi).to(dev), torch.from_numpy(wl.log_A).to(dev)
    ll = torch.from_numpy(wl.log_lik).to(dev)
    bes = [LibBackend() for _ in range(world)]
    sl = _slices(wl.T, world)
    aggs, infos = [], []
    for r, (t0, n) in enumerate(sl):
        a, i = bes[r].smooth_reduce(lp, la, ll[t0:t0 + n], t0)
        aggs.append(a); infos.append(i)
    agg_all = torch.cat(aggs)
    outs = [bes[r].smooth_finish(lp, la, ll[t0:t0 + n], t0, agg_all, r, world) for r, (t0, n) in enumerate(sl)]
    torch.cuda.synchronize()
    filt = torch.cat([o[0] for o in outs]).cpu().numpy()
    sm = torch.cat([o[1] for o in outs]).cpu().numpy()
    lz = sum(float(o[2].item()) for o in outs)
    info = [int(i.item()) for i in infos] + [int(o[3].item()) for o in outs]
    return filt, sm, lz, info


def emulate_viterbi(wl, world):
    from paper_2102_05743_b200.dist import LibBackend
    dev = torch.device("cuda")
    lp, la = torch.from_numpy(wl.log_pi).to(dev), torch.from_numpy(wl.log_A).to(dev)
    ll = torch.from_numpy(wl.log_lik).to(dev)
    bes = [LibBackend() for _ in range(world)]
    sl = _slices(wl.T, world)
    agg_all = torch.cat([bes[r].viterbi_reduce(lp, la, ll[t0:t0 + n], t0)[0] for r, (t0, n) in enumerate(sl)])
    fw = [bes[r].viterbi_forward(lp, la, ll[t0:t0 + n], t0, agg_all, r, world) for r, (t0, n) in enumerate(sl)]
    rec_all = torch.cat([f[0] for f in fw])
    fin = [bes[r].viterbi_finish(lp, la, ll[t0:t0 + n], t0, rec_all, r, world) for r, (t0, n) in enumerate(sl)]
    torch.cuda.synchronize()
    path = torch.cat([f[0] for f in fin]).cpu().numpy()
    lpr = sum(float(f[1].item()) for f in fw)
    info = [int(f[2].item()) for f in fw] + [int(f[1].item()) for f in fin]
    return path, lpr, info


@pytest.mark.parametrize("world,T", [(1, 100_000), (2, 1_000_000), (4, 1_000_003), (8, 2_000_000), (3, 5000),
                                     (8, 64), (8, 8)])
def test_dist_smoother_rank_invariance(world, T):
    wl = W.ge(T, seed=5)
    filt, sm, lz, info = emulate_smooth(wl, world)
    assert all(i == 0 for i in info)
    o = oracle.smooth(wl.log_pi, wl.log_A, wl.log_lik)
    assert float(np.abs(sm - o["smoothed"]).max()) <= TOL_MARG
    assert float(np.abs(filt - o["filtered"]).max()) <= TOL_MARG
    assert rel(lz, o["log_z"]) <= TOL_REL


@pytest.mark.parametrize("world,T", [(1, 50_000), (2, 1_000_000), (4, 999_999), (8, 2_000_000), (3, 5000), (8, 64)])
def test_dist_viterbi_rank_invariance(world, T):
    wl = W.ge(T, seed=6, jitter=0.1)
    path, lpr, info = emulate_viterbi(wl, world)
    assert all(i == 0 for i in info)
    v = oracle.viterbi(wl.log_pi, wl.log_A, wl.log_lik)
    assert rel(lpr, v["log_prob"]) <= TOL_REL
    _, gap = oracle.max_marginals(wl.log_pi, wl.log_A, wl.log_lik)
    safe = gap >= TAU
    assert int(((path != v["path"]) & safe).sum()) == 0
    jw = oracle.joint_weight(wl.log_pi, wl.log_A, wl.log_lik, path)
    assert rel(jw, v["log_prob"]) <= TOL_REL


def test_dist_planted_path_exact():
    wl = W.planted(5, 300_000, seed=4)
    path, lpr, info = emulate_viterbi(wl, 4)
    assert np.array_equal(path, wl.states)


def test_dist_info_global_step():
    wl = W.ge(400_000, seed=9)
    wl.log_lik[250_123, :] = -np.inf
    _, _, _, info = emulate_smooth(wl, 4)
    assert min(i for i in info if i > 0) == 250_124
    _, _, vinfo = emulate_viterbi(wl, 4)
    assert min(i for i in vinfo if i > 0) == 250_124


@pytest.mark.parametrize("world", [1, 3, 8])
@pytest.mark.parametrize("codes", [(0, 0, 0, 0), (0, 17, 0, 5), (-1, 3, 0, 0), (0, 0, 9, -1)])
def test_dist_pack_combine(world, codes):
    """hmm_dist_pack / hmm_dist_combine against the tensor-op combination they replace: records in rank
    order, log Z and log_prob summed in rank order from 0.0 (bit for bit), global info codes."""
    from paper_2102_05743_b200.dist import LibBackend
    be = LibBackend()
    dev = torch.device("cuda")
    g = torch.Generator().manual_seed(world * 31 + codes[1])
    rows, recs, lzs, lps, infos = [], [], [], [], []
    for r in range(world):
        rec = torch.randint(0, 256, (16,), dtype=torch.uint8, generator=g)
        lz = torch.randn(1, dtype=torch.float64, generator=g) * 1e6
        lp = torch.randn(1, dtype=torch.float64, generator=g) * 1e6
        cs = [c if r == world - 1 or c <= 0 else c + 100 * r for c in codes]  # rank 0 holds the smallest
        ii = [torch.tensor([c], dtype=torch.int32) for c in cs]
        rows.append(be.pack(rec.to(dev), lz.to(dev), lp.to(dev), *[t.to(dev) for t in ii]))
        recs.append(rec); lzs.append(lz); lps.append(lp); infos.append(cs)
    gathered = torch.cat(rows)
    rec_all, lz, lp, info, vinfo = be.combine(gathered, world)
    torch.cuda.synchronize()
    assert torch.equal(rec_all.cpu(), torch.cat(recs))
    ez, ep = torch.zeros(1, dtype=torch.float64), torch.zeros(1, dtype=torch.float64)
    for r in range(world):
        ez += lzs[r]
        ep += lps[r]
    assert float(lz[0]) == float(ez[0]) and float(lp[0]) == float(ep[0])
    s_codes = [c for cs in infos for c in cs[:2]]
    v_codes = [c for cs in infos for c in cs[2:]]
    assert int(info[0]) == _expected_info(s_codes)
    assert int(vinfo[0]) == _expected_info(v_codes)


def _expected_info(codes):
    """hmmscan.h: -1 if any rank reported -1, else the smallest positive code, else 0."""
    if -1 in codes:
        return -1
    pos = [c for c in codes if c > 0]
    return min(pos) if pos else 0


def test_dist_pack_null_inputs_are_zero():
    """hmm_dist_pack: NULL inputs contribute zeros (the smoother-only and Viterbi-only steps)."""
    from paper_2102_05743_b200.dist import LibBackend
    be = LibBackend()
    dev = torch.device("cuda")
    lz = torch.tensor([-123.5], dtype=torch.float64, device=dev)
    i1 = torch.tensor([7], dtype=torch.int32, device=dev)
    row = be.pack(None, lz, None, i1, None, None, None)
    torch.cuda.synchronize()
    assert row.cpu().tolist() == [0.0, 0.0, -123.5, 0.0, 7.0, 0.0, 0.0, 0.0]
    rec_all, z, p, info, vinfo = be.combine(torch.cat([row, row]), 2)
    assert float(z[0]) == -247.0 and float(p[0]) == 0.0 and int(info[0]) == 7 and int(vinfo[0]) == 0


def test_dist_misaligned_output_rejected():
    """Split phase: all phases of a rank run the kernel chosen from log_lik's alignment, so a finish
    output that is not 16-B aligned is an error instead of a silent switch of kernel (hmmscan.h)."""
    import ctypes
    from paper_2102_05743_b200 import _ptr, _stream
    from paper_2102_05743_b200.dist import LibBackend
    be = LibBackend()
    wl = W.ge(10_000, seed=3)
    dev = torch.device("cuda")
    lp, la = torch.from_numpy(wl.log_pi).to(dev), torch.from_numpy(wl.log_A).to(dev)
    ll = torch.from_numpy(wl.log_lik).to(dev)
    agg, _ = be.smooth_reduce(lp, la, ll, 0)
    ws = be.ws(0, 4, wl.T, dev)
    big = torch.empty(wl.T * 4 + 1, dtype=torch.float32, device=dev)
    lzp = torch.empty(1, dtype=torch.float64, device=dev)
    info = torch.empty(1, dtype=torch.int32, device=dev)
    st = be.L.hmm_smooth_dist_finish(4, wl.T, 0, _ptr(lp), _ptr(la), _ptr(ll), _ptr(agg), 0, 1,
                                     ctypes.c_void_p(big.data_ptr() + 4), _ptr(big), _ptr(lzp), _ptr(info),
                                     _ptr(ws), ws.numel(), _stream(None))
    assert st == 1
    f, s, z, i = be.smooth_finish(lp, la, ll, 0, agg, 0, 1)  # the workspace is still consistent
    torch.cuda.synchronize()
    assert int(i[0]) == 0


@pytest.mark.parametrize("D,world,T", [(12, 2, 20_000), (16, 4, 100_003), (24, 3, 50_000), (40, 8, 100_000),
                                       (64, 2, 100_000), (64, 1, 5000), (33, 8, 64)])
def test_dist_smoother_large_D(D, world, T):
    """Split-phase smoother at D > 8 (the large-D block scan: reduce -> DP x DP rank aggregate, finish ->
    rank carries, carry chains, sweeps): rank-count invariant and equal to the oracle on the whole
    sequence (D = 64 runs the tcgen05 leaf products)."""
    wl = W.dense(D, T, seed=7 + D)
    filt, sm, lz, info = emulate_smooth(wl, world)
    assert all(i == 0 for i in info), info
    o = oracle.smooth(wl.log_pi, wl.log_A, wl.log_lik)
    assert float(np.abs(sm - o["smoothed"]).max()) <= TOL_MARG
    assert float(np.abs(filt - o["filtered"]).max()) <= TOL_MARG
    assert rel(lz, o["log_z"]) <= TOL_REL


def test_dist_large_D_info():
    wl = W.dense(20, 30_000, seed=3)
    wl.log_lik[17_345, :] = -np.inf
    filt, sm, lz, info = emulate_smooth(wl, 4)
    assert 17_346 in info  # the first impossible GLOBAL step + 1, reported by the rank that holds it
    path, lpr, vinfo = emulate_viterbi(wl, 4)
    assert 17_346 in vinfo


@pytest.mark.parametrize("D,world,T", [(12, 2, 20_000), (16, 4, 100_003), (24, 3, 50_000), (40, 8, 100_000),
                                       (64, 2, 100_000), (64, 1, 5000), (33, 8, 64)])
def test_dist_viterbi_large_D(D, world, T):
    """Split-phase Viterbi at D > 8 (records = DP-byte rank maps + x*): the MAP path is bit-exact where the
    oracle's max-marginal gap >= TAU and attains the MAP weight; log_prob to 1e-6."""
    wl = W.dense(D, T, seed=11 + D)
    wl.log_lik = wl.log_lik + W.random_potentials(D, T, seed=5, sigma=0.1).log_lik
    path, lpr, info = emulate_viterbi(wl, world)
    assert all(i == 0 for i in info), info
    v = oracle.viterbi(wl.log_pi, wl.log_A, wl.log_lik)
    assert rel(lpr, v["log_prob"]) <= TOL_REL
    _, gap = oracle.max_marginals(wl.log_pi, wl.log_A, wl.log_lik)
    safe = gap >= TAU
    assert np.array_equal(path[safe], v["path"][safe])
    assert rel(oracle.joint_weight(wl.log_pi, wl.log_A, wl.log_lik, path), v["log_prob"]) <= TOL_REL


@pytest.mark.parametrize("D", [4, 20])
def test_dist_python_orchestration_one_rank(D):
    """paper_2102_05743_b200.dist.smooth_viterbi_dist / viterbi_dist end to end in a one-rank gloo group on
    the GPU (the collectives degenerate to copies): covers the 16-byte-record path (D <= 8, packed with
    the scalars) and the wide-record path (D > 8, its own all-gather)."""
    import os
    import torch.distributed as dist
    from paper_2102_05743_b200 import dist as HD
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29613")
        dist.init_process_group("gloo", rank=0, world_size=1)
    wl = W.dense(D, 20_000, seed=21 + D)
    wl.log_lik = wl.log_lik + W.random_potentials(D, 20_000, seed=8, sigma=0.1).log_lik
    dev = torch.device("cuda")
    lp, la, ll = (torch.from_numpy(x).to(dev) for x in (wl.log_pi, wl.log_A, wl.log_lik))
    f, s, lz, info, path, lpr, vinfo = HD.smooth_viterbi_dist(lp, la, ll, 0)
    p2, lpr2, vinfo2 = HD.viterbi_dist(lp, la, ll, 0)
    torch.cuda.synchronize()
    o = oracle.smooth(wl.log_pi, wl.log_A, wl.log_lik)
    v = oracle.viterbi(wl.log_pi, wl.log_A, wl.log_lik)
    assert int(info.item()) == 0 and int(vinfo.item()) == 0 and int(vinfo2.item()) == 0
    assert float(np.abs(s.cpu().numpy() - o["smoothed"]).max()) <= TOL_MARG
    assert rel(float(lz.item()), o["log_z"]) <= TOL_REL
    for p_, l_ in ((path, lpr), (p2, lpr2)):
        assert rel(float(l_.item()), v["log_prob"]) <= TOL_REL
        assert rel(oracle.joint_weight(wl.log_pi, wl.log_A, wl.log_lik, p_.cpu().numpy()), v["log_prob"]) <= TOL_REL
