"""Split-phase multi-GPU path: one HMM sequence partitioned along T across the ranks of a process group.

Rank r owns the contiguous global steps [t_base, t_base + T_local) (``partition``).  The exchange is
the only collective of the method: every rank reduces its slice to one D x D
aggregate (the ordered product of its elements, Def. 3 / Def. 5 of the paper), the W aggregates are
all-gathered (NCCL over NVLink on B200s; ~W*80 bytes at D=4), and every rank runs a local finish
pass with carries folded from the gathered aggregates in rank order.  log Z / log_prob are the
fixed-order sums of per-rank partials (a second tiny all-gather), so every rank holds bitwise-identical
scalars.  Viterbi adds one more tiny all-gather of the rank backpointer maps (D bytes + x*).
This module holds no arithmetic of the method: partitioning, collectives and marshalling only; the
scalar combination (rank-order sums, info codes) runs in the library (hmm_dist_pack / hmm_dist_combine).

The compute is done by ``LibBackend`` (the C ABI of libhmmscan.so).  The orchestration takes the
backend as a parameter so its host logic can be exercised on CPU with gloo (tests/test_dist_gloo.py).
"""
from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from . import HmmError, _check, _ptr, _stream, lib

RECORD_BYTES = 16


class _nvtx:
    """NVTX range around a phase (visible in nsys / ncu timelines; a host-side marker, no device work)."""

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        torch.cuda.nvtx.range_push(self.name)

    def __exit__(self, *a):
        torch.cuda.nvtx.range_pop()


def partition(T: int, world: int, rank: int, align: int = 8) -> tuple[int, int]:
    """Contiguous slices with boundaries on multiples of `align` (16-B aligned slices for the bulk
    copies); if that would leave a rank empty, an unaligned equal split.  Returns (t_base, T_local)."""
    if T < world:
        raise HmmError("need T >= world")
    per = -(-T // world)
    per = -(-per // align) * align
    if per * (world - 1) >= T:  # some rank would be empty: equal split for everyone
        return rank * T // world, (rank + 1) * T // world - rank * T // world
    t0 = rank * per
    return t0, min(per, T - t0)


class LibBackend:
    """Device compute of the phases through the C ABI (hmmscan.h split-phase entry points)."""

    def __init__(self):
        L = lib()
        i32, i64, p, sz = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t
        L.hmm_dist_agg_bytes.restype = sz
        L.hmm_dist_agg_bytes.argtypes = [i32]
        L.hmm_dist_record_bytes_d.restype = sz
        L.hmm_dist_record_bytes_d.argtypes = [i32]
        L.hmm_dist_workspace_size.restype = sz
        L.hmm_dist_workspace_size.argtypes = [i32, i32, i64]
        L.hmm_smooth_dist_reduce.argtypes = [i32, i64, i64, p, p, p, p, p, p, sz, p]
        L.hmm_smooth_dist_finish.argtypes = [i32, i64, i64, p, p, p, p, i32, i32, p, p, p, p, p, sz, p]
        L.hmm_viterbi_dist_reduce.argtypes = [i32, i64, i64, p, p, p, p, p, p, sz, p]
        L.hmm_viterbi_dist_forward.argtypes = [i32, i64, i64, p, p, p, p, i32, i32, p, p, p, p, sz, p]
        L.hmm_viterbi_dist_finish.argtypes = [i32, i64, i64, p, p, p, p, i32, i32, p, p, p, sz, p]
        L.hmm_dist_pack.argtypes = [p, p, p, p, p, p, p, p, p]
        L.hmm_dist_combine.argtypes = [i32, p, p, p, p, p, p, p]
        for f in ("hmm_smooth_dist_reduce", "hmm_smooth_dist_finish", "hmm_viterbi_dist_reduce",
                  "hmm_viterbi_dist_forward", "hmm_viterbi_dist_finish", "hmm_dist_pack", "hmm_dist_combine"):
            getattr(L, f).restype = i32
        self.L = L
        self._ws = {}

    def pack(self, rec, lzp, lpp, s_i1, s_i2, v_i1, v_i2):
        """One rank's 8-double scalar record (hmm_dist_pack); None inputs contribute zeros."""
        dev = next(x for x in (rec, lzp, lpp, s_i1, s_i2, v_i1, v_i2) if x is not None).device
        out = torch.empty(8, dtype=torch.float64, device=dev)
        _check(self.L.hmm_dist_pack(_ptr(rec), _ptr(lzp), _ptr(lpp), _ptr(s_i1), _ptr(s_i2), _ptr(v_i1), _ptr(v_i2),
                                    _ptr(out), _stream(None)), "hmm_dist_pack")
        return out

    def combine(self, g, world):
        """From the gathered records (hmm_dist_combine): the Viterbi rank records in rank order, log Z and
        log_prob (sums of the partials in rank order) and the global info codes of both operations."""
        dev = g.device
        rec_all = torch.empty(16 * world, dtype=torch.uint8, device=dev)
        lz = torch.empty(1, dtype=torch.float64, device=dev)
        lp = torch.empty(1, dtype=torch.float64, device=dev)
        info = torch.empty(1, dtype=torch.int32, device=dev)
        vinfo = torch.empty(1, dtype=torch.int32, device=dev)
        _check(self.L.hmm_dist_combine(world, _ptr(g), _ptr(rec_all), _ptr(lz), _ptr(lp), _ptr(info), _ptr(vinfo),
                                       _stream(None)), "hmm_dist_combine")
        return rec_all, lz, lp, info, vinfo

    def agg_bytes(self, D):
        return int(self.L.hmm_dist_agg_bytes(D))

    def ws(self, op, D, T_local, device):
        key = (op, D, T_local, device)
        if key not in self._ws:
            n = int(self.L.hmm_dist_workspace_size(op, D, T_local))
            if n == 0:
                raise HmmError(f"split phase unsupported for D={D}")
            self._ws[key] = torch.zeros(n, dtype=torch.uint8, device=device)
        return self._ws[key]

    def smooth_reduce(self, lp, la, ll, t_base):
        T, D = ll.shape
        ws = self.ws(0, D, T, ll.device)
        agg = torch.empty(self.agg_bytes(D), dtype=torch.uint8, device=ll.device)
        info = torch.empty(1, dtype=torch.int32, device=ll.device)
        _check(self.L.hmm_smooth_dist_reduce(D, T, t_base, _ptr(lp), _ptr(la), _ptr(ll), _ptr(agg), _ptr(info),
                                             _ptr(ws), ws.numel(), _stream(None)), "hmm_smooth_dist_reduce")
        return agg, info

    def smooth_finish(self, lp, la, ll, t_base, agg_all, rank, world):
        T, D = ll.shape
        ws = self.ws(0, D, T, ll.device)
        filt, sm = torch.empty_like(ll), torch.empty_like(ll)
        lzp = torch.empty(1, dtype=torch.float64, device=ll.device)
        info = torch.empty(1, dtype=torch.int32, device=ll.device)
        _check(self.L.hmm_smooth_dist_finish(D, T, t_base, _ptr(lp), _ptr(la), _ptr(ll), _ptr(agg_all), rank, world,
                                             _ptr(filt), _ptr(sm), _ptr(lzp), _ptr(info), _ptr(ws), ws.numel(),
                                             _stream(None)), "hmm_smooth_dist_finish")
        return filt, sm, lzp, info

    def viterbi_reduce(self, lp, la, ll, t_base):
        T, D = ll.shape
        ws = self.ws(1, D, T, ll.device)
        agg = torch.empty(self.agg_bytes(D), dtype=torch.uint8, device=ll.device)
        info = torch.empty(1, dtype=torch.int32, device=ll.device)
        _check(self.L.hmm_viterbi_dist_reduce(D, T, t_base, _ptr(lp), _ptr(la), _ptr(ll), _ptr(agg), _ptr(info),
                                              _ptr(ws), ws.numel(), _stream(None)), "hmm_viterbi_dist_reduce")
        return agg, info

    def viterbi_forward(self, lp, la, ll, t_base, agg_all, rank, world):
        T, D = ll.shape
        ws = self.ws(1, D, T, ll.device)
        rec = torch.zeros(int(self.L.hmm_dist_record_bytes_d(D)), dtype=torch.uint8, device=ll.device)
        lpp = torch.empty(1, dtype=torch.float64, device=ll.device)
        info = torch.empty(1, dtype=torch.int32, device=ll.device)
        _check(self.L.hmm_viterbi_dist_forward(D, T, t_base, _ptr(lp), _ptr(la), _ptr(ll), _ptr(agg_all), rank, world,
                                               _ptr(rec), _ptr(lpp), _ptr(info), _ptr(ws), ws.numel(),
                                               _stream(None)), "hmm_viterbi_dist_forward")
        return rec, lpp, info

    def viterbi_finish(self, lp, la, ll, t_base, rec_all, rank, world):
        T, D = ll.shape
        ws = self.ws(1, D, T, ll.device)
        path = torch.empty(T, dtype=torch.int32, device=ll.device)
        info = torch.empty(1, dtype=torch.int32, device=ll.device)
        _check(self.L.hmm_viterbi_dist_finish(D, T, t_base, _ptr(lp), _ptr(la), _ptr(ll), _ptr(rec_all), rank, world,
                                              _ptr(path), _ptr(info), _ptr(ws), ws.numel(), _stream(None)),
               "hmm_viterbi_dist_finish")
        return path, info


_default = None


def _backend(backend):
    global _default
    if backend is not None:
        return backend
    if _default is None:
        _default = LibBackend()
    return _default


def _all_gather(x: torch.Tensor, group=None) -> torch.Tensor:
    """Rank-ordered concatenation of a small per-rank tensor (NCCL: all_gather_into_tensor)."""
    world = dist.get_world_size(group)
    if x.is_cuda and dist.get_backend(group) == "nccl":
        out = torch.empty(world * x.numel(), dtype=x.dtype, device=x.device)
        dist.all_gather_into_tensor(out, x.contiguous().view(-1), group=group)
        return out
    xc = x.detach().cpu().contiguous()  # gloo (CPU tests / single-GPU multi-process smoke runs)
    parts = [torch.empty_like(xc) for _ in range(world)]
    dist.all_gather(parts, xc, group=group)
    return torch.cat([q.view(-1) for q in parts]).to(x.device)


def smooth_dist(log_pi, log_A, log_lik_local, t_base: int, group=None, backend=None):
    """Parallel smoother over a T-partitioned sequence (1 <= D <= 64).  Returns (filtered, smoothed, log_z [1], info [1])
    for the local slice; log_z and info are global and identical on every rank (rank-order sums and
    info combination done by the library's hmm_dist_combine)."""
    be = _backend(backend)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    agg, info1 = be.smooth_reduce(log_pi, log_A, log_lik_local, t_base)
    agg_all = _all_gather(agg, group)                       # the method's one exchange step
    filt, sm, lzp, info2 = be.smooth_finish(log_pi, log_A, log_lik_local, t_base, agg_all, rank, world)
    g = _all_gather(be.pack(None, lzp, None, info1, info2, None, None), group)
    _, log_z, _, info, _ = be.combine(g, world)
    return filt, sm, log_z, info


def viterbi_dist(log_pi, log_A, log_lik_local, t_base: int, group=None, backend=None):
    """Parallel MAP path over a T-partitioned sequence.  Returns (path of the local slice, log_prob [1],
    info [1]); log_prob and info are global.  Two all-gathers: the rank aggregates, then the rank records
    (backpointer map + x*) together with the log_prob partials and info codes."""
    be = _backend(backend)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    agg, info1 = be.viterbi_reduce(log_pi, log_A, log_lik_local, t_base)
    agg_all = _all_gather(agg, group)
    rec, lpp, info2 = be.viterbi_forward(log_pi, log_A, log_lik_local, t_base, agg_all, rank, world)
    if rec.numel() == RECORD_BYTES:
        g = _all_gather(be.pack(rec, None, lpp, None, None, info1, info2), group)
        rec_all, _, log_prob, _, info = be.combine(g, world)
    else:  # D > 8: the wider rank records travel in their own all-gather
        rec_all = _all_gather(rec, group)
        g = _all_gather(be.pack(None, None, lpp, None, None, info1, info2), group)
        _, _, log_prob, _, info = be.combine(g, world)
    # finish only backtracks: its info is always 0 (errors are reported by reduce / forward, hmmscan.h)
    path, _ = be.viterbi_finish(log_pi, log_A, log_lik_local, t_base, rec_all, rank, world)
    return path, log_prob, info


def smooth_viterbi_dist(log_pi, log_A, log_lik_local, t_base: int, group=None, backend=None):
    """Smoother and MAP path of the same T-partitioned sequence with the collectives of both merged:
    two all-gathers per call instead of four (the rank aggregates of both semirings together; then the
    Viterbi rank records together with every scalar partial).  Returns
    (filtered, smoothed, log_z [1], info [1], path, log_prob [1], vinfo [1]) for the local slice."""
    be = _backend(backend)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    with _nvtx("hmm.reduce"):
        s_agg, s_i1 = be.smooth_reduce(log_pi, log_A, log_lik_local, t_base)
        v_agg, v_i1 = be.viterbi_reduce(log_pi, log_A, log_lik_local, t_base)
    na = s_agg.numel()
    with _nvtx("hmm.allgather.aggregates"):
        both = _all_gather(torch.cat([s_agg.view(-1), v_agg.view(-1)]), group).view(world, 2 * na)
    s_all = both[:, :na].contiguous().view(-1)
    v_all = both[:, na:].contiguous().view(-1)
    with _nvtx("hmm.finish"):
        filt, sm, lzp, s_i2 = be.smooth_finish(log_pi, log_A, log_lik_local, t_base, s_all, rank, world)
        rec, lpp, v_i2 = be.viterbi_forward(log_pi, log_A, log_lik_local, t_base, v_all, rank, world)
    with _nvtx("hmm.allgather.records"):
        if rec.numel() == RECORD_BYTES:
            g = _all_gather(be.pack(rec, lzp, lpp, s_i1, s_i2, v_i1, v_i2), group)
            rec_all, log_z, log_prob, info, vinfo = be.combine(g, world)
        else:  # D > 8: the wider rank records travel in their own all-gather
            rec_all = _all_gather(rec, group)
            g = _all_gather(be.pack(None, lzp, lpp, s_i1, s_i2, v_i1, v_i2), group)
            _, log_z, log_prob, info, vinfo = be.combine(g, world)
    with _nvtx("hmm.backtrack"):
        path, _ = be.viterbi_finish(log_pi, log_A, log_lik_local, t_base, rec_all, rank, world)
    return filt, sm, log_z, info, path, log_prob, vinfo
