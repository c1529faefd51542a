"""Multi-process host logic of the split-phase path on CPU (gloo, world sizes 2 and 3).

paper_2102_05743_b200.dist owns partitioning, the all-gathers and the fixed-order reductions; the
per-rank compute goes through a backend.  Here a test double (`NumpyBackend`, fp64, written in this
file) stands in for the CUDA library so the orchestration can run without a GPU; the results of the
whole W-rank pipeline must match the fp64 oracle on the unpartitioned sequence.  (The real kernels'
phases are covered by tests/test_gpu_dist.py on one GPU.)
"""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as W


class NumpyBackend:
    """fp64 reference of the four phases with the library's record semantics (test double)."""

    def _elems(self, lp, la, ll, t_base):
        A = np.exp(la.numpy().astype(np.float64)); pi = np.exp(lp.numpy().astype(np.float64))
        L = ll.numpy().astype(np.float64)
        m = L.max(1, keepdims=True)
        return A, pi, np.exp(L - m), m[:, 0]

    def smooth_reduce(self, lp, la, ll, t_base):
        A, pi, l, _ = self._elems(lp, la, ll, t_base)
        D = A.shape[0]
        P = np.eye(D)
        for i in range(l.shape[0]):
            E = (np.tile(pi, (D, 1)) if t_base + i == 0 else A) * l[i][None, :]
            P = P @ E
            P /= P.max()
        return torch.from_numpy(P.reshape(-1).copy()).view(torch.uint8), torch.zeros(1, dtype=torch.int32)

    def smooth_finish(self, lp, la, ll, t_base, agg_all, rank, world):
        A, pi, l, m = self._elems(lp, la, ll, t_base)
        D = A.shape[0]
        aggs = agg_all.view(torch.float64).numpy().reshape(world, D, D)
        pre = np.ones(D) / D
        for q in range(rank):
            pre = pre @ aggs[q]; pre /= pre.sum()
        suf = np.ones(D)
        for q in range(world - 1, rank, -1):
            suf = aggs[q] @ suf; suf /= suf.max()
        n = l.shape[0]
        alpha = np.zeros((n, D)); a = pre / pre.sum(); lz = 0.0
        for i in range(n):
            ah = pi * l[i] if t_base + i == 0 else (a @ A) * l[i]
            c = ah.sum(); a = ah / c; alpha[i] = a; lz += np.log(c) + m[i]
        sm = np.zeros((n, D)); b = suf
        for i in range(n - 1, -1, -1):
            g = alpha[i] * b; sm[i] = g / g.sum()
            b = A @ (l[i] * b); b /= b.max()
        f32 = lambda x: torch.from_numpy(x.astype(np.float32))
        return f32(alpha), f32(sm), torch.tensor([lz], dtype=torch.float64), torch.zeros(1, dtype=torch.int32)

    def viterbi_reduce(self, lp, la, ll, t_base):
        LA = la.numpy().astype(np.float64); LP = lp.numpy().astype(np.float64); L = ll.numpy().astype(np.float64)
        D = LA.shape[0]
        P = np.where(np.eye(D) > 0, 0.0, -np.inf)
        for i in range(L.shape[0]):
            E = (np.tile(LP, (D, 1)) if t_base + i == 0 else LA) + L[i][None, :]
            P = (P[:, :, None] + E[None, :, :]).max(1)
            P -= P.max()
        return torch.from_numpy(P.reshape(-1).copy()).view(torch.uint8), torch.zeros(1, dtype=torch.int32)

    def viterbi_forward(self, lp, la, ll, t_base, agg_all, rank, world):
        LA = la.numpy().astype(np.float64); LP = lp.numpy().astype(np.float64); L = ll.numpy().astype(np.float64)
        D = LA.shape[0]
        aggs = agg_all.view(torch.float64).numpy().reshape(world, D, D)
        V = np.zeros(D)
        for q in range(rank):
            V = (V[:, None] + aggs[q]).max(0); V -= V.max()
        lp_part = 0.0
        orig = np.arange(D)
        self.bp = []
        for i in range(L.shape[0]):
            E = (np.tile(LP, (D, 1)) if t_base + i == 0 else LA)
            S = V[:, None] + E
            u = S.argmax(0)
            Vn = S.max(0) + L[i]
            o = Vn.max(); lp_part += o; V = Vn - o
            self.bp.append(u); orig = orig[u]
        xs = int(np.argmax(V == 0.0))
        rec = np.zeros(16, np.uint8)
        rec[:D] = orig.astype(np.uint8)
        rec[8:12] = np.frombuffer(np.int32(xs).tobytes(), np.uint8)
        return torch.from_numpy(rec), torch.tensor([lp_part], dtype=torch.float64), torch.zeros(1, dtype=torch.int32)

    def pack(self, rec, lzp, lpp, s_i1, s_i2, v_i1, v_i2):
        """hmm_dist_pack's record layout: 2 doubles of Viterbi record, log Z / log_prob partials, 4 codes."""
        out = np.zeros(8)
        if rec is not None:
            out[:2] = rec.numpy().view(np.float64)
        for k, x in ((2, lzp), (3, lpp), (4, s_i1), (5, s_i2), (6, v_i1), (7, v_i2)):
            if x is not None:
                out[k] = float(x.reshape(-1)[0])
        return torch.from_numpy(out)

    def combine(self, g, world):
        """hmm_dist_combine: records in rank order, partial sums in rank order from 0.0, info codes."""
        G = g.numpy().reshape(world, 8)
        rec_all = torch.from_numpy(np.ascontiguousarray(G[:, :2]).view(np.uint8).reshape(-1).copy())
        lz = 0.0
        lp = 0.0
        for r in range(world):
            lz += G[r, 2]
            lp += G[r, 3]

        def codes(c0):
            cs = [int(c) for c in G[:, c0:c0 + 2].reshape(-1)]
            if -1 in cs:
                return -1
            pos = [c for c in cs if c > 0]
            return min(pos) if pos else 0
        i32 = lambda v: torch.tensor([v], dtype=torch.int32)
        return (rec_all, torch.tensor([lz], dtype=torch.float64), torch.tensor([lp], dtype=torch.float64),
                i32(codes(4)), i32(codes(6)))

    def viterbi_finish(self, lp, la, ll, t_base, rec_all, rank, world):
        recs = rec_all.numpy().reshape(world, 16)
        x = int(np.frombuffer(recs[world - 1, 8:12].tobytes(), np.int32)[0])
        for q in range(world - 1, rank, -1):
            x = int(recs[q, x])
        n = ll.shape[0]
        path = np.zeros(n, np.int32)
        for i in range(n - 1, -1, -1):
            path[i] = x; x = int(self.bp[i][x])
        return torch.from_numpy(path), torch.zeros(1, dtype=torch.int32)


def _worker(rank, world, port, T, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2102_05743_b200 import dist as HD
    wl = W.ge(T, seed=21, jitter=0.1)
    t0, n = HD.partition(T, world, rank)
    ll = torch.from_numpy(np.ascontiguousarray(wl.log_lik[t0:t0 + n]))
    lp, la = torch.from_numpy(wl.log_pi), torch.from_numpy(wl.log_A)
    be = NumpyBackend()
    filt, sm, lz, info = HD.smooth_dist(lp, la, ll, t0, backend=be)
    path, lpr, vinfo = HD.viterbi_dist(lp, la, ll, t0, backend=be)
    # the merged-collective variant returns the same values
    f2, s2, lz2, i2, p2, lp2, vi2 = HD.smooth_viterbi_dist(lp, la, ll, t0, backend=be)
    assert torch.equal(s2, sm) and torch.equal(f2, filt) and torch.equal(p2, path)
    assert float(lz2[0]) == float(lz[0]) and float(lp2[0]) == float(lpr[0])
    assert int(i2[0]) == int(info[0]) and int(vi2[0]) == int(vinfo[0])
    np.savez(os.path.join(outdir, f"r{rank}.npz"), t0=t0, filt=filt.numpy(), sm=sm.numpy(), lz=lz.numpy(),
             info=info.numpy(), path=path.numpy(), lpr=lpr.numpy(), vinfo=vinfo.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world,T", [(2, 2001), (3, 1000)])
def test_split_phase_orchestration_gloo(world, T):
    import oracle
    from paper_2102_05743_b200 import dist as HD
    port = 29500 + (os.getpid() % 2000) + world
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, port, T, d), nprocs=world, join=True)
        res = [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(world)]
    wl = W.ge(T, seed=21, jitter=0.1)
    o = oracle.smooth(wl.log_pi, wl.log_A, wl.log_lik)
    v = oracle.viterbi(wl.log_pi, wl.log_A, wl.log_lik)
    # the partition tiles [0, T) in rank order
    assert [int(r["t0"]) for r in res] == [HD.partition(T, world, q)[0] for q in range(world)]
    sm = np.concatenate([r["sm"] for r in res]); filt = np.concatenate([r["filt"] for r in res])
    path = np.concatenate([r["path"] for r in res])
    assert sm.shape == (T, 4)
    np.testing.assert_allclose(sm, o["smoothed"], atol=1e-6)
    np.testing.assert_allclose(filt, o["filtered"], atol=1e-6)
    for r in res:  # global scalars identical on every rank
        assert r["lz"][0] == res[0]["lz"][0] and r["lpr"][0] == res[0]["lpr"][0]
        assert int(r["info"][0]) == 0 and int(r["vinfo"][0]) == 0
    assert abs(res[0]["lz"][0] - o["log_z"]) < 1e-8 * abs(o["log_z"])
    assert abs(res[0]["lpr"][0] - v["log_prob"]) < 1e-8 * abs(v["log_prob"])
    assert np.array_equal(path, v["path"])


def test_partition_properties():
    from paper_2102_05743_b200.dist import partition
    for T in [8, 9, 100, 1001, 10**6 + 3]:
        for world in [1, 2, 3, 8]:
            if T < world:
                continue
            parts = [partition(T, world, r) for r in range(world)]
            assert parts[0][0] == 0
            assert sum(n for _, n in parts) == T
            for (a, n), (b, _) in zip(parts, parts[1:]):
                assert a + n == b
            assert all(n >= 1 for _, n in parts)
