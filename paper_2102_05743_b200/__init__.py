"""paper_2102_05743_b200 — B200-native temporally parallel HMM inference (Hassan, Särkkä,
García-Fernández, "Temporal Parallelization of Inference in Hidden Markov Models", arXiv 2102.05743).

Thin Python binding over the C ABI of ``lib/libhmmscan.so`` (``include/hmmscan.h``): argument
marshalling only — every step of the hot path runs in the library's sm_100a kernels.  PyTorch is used
for device memory and streams.  There is no CPU fallback: importing works anywhere, but every compute
call requires the CUDA library and a CUDA device and raises otherwise.

    filtered, smoothed, log_z, info = smooth(log_pi, log_A, log_lik)       # Algorithm 3
    path, log_prob, info = viterbi(log_pi, log_A, log_lik)                  # Def. 5 + backpointers

``log_lik`` is [T, D] (single sequence) or [B, T, D] (batched, shared log_pi / log_A).
"""
from __future__ import annotations

import ctypes
import os
import re

import torch

from .build import LIB, ROOT

HMM_OP_SMOOTH, HMM_OP_VITERBI, HMM_OP_SMOOTH_STATS = 0, 1, 2
HMM_OP_VITERBI_MAXPRODUCT, HMM_OP_VITERBI_PATHELEM = 5, 6
HMM_OP_SMOOTH_VARLEN, HMM_OP_VITERBI_VARLEN = 7, 8
HMM_INFO_BAD_LENGTH = -4
HMM_INFO_AMBIGUOUS, HMM_INFO_NO_PATH = -2, -3
HMM_PATHELEM_MAX_T = 1024
HMM_MAX_D = 64
STATUS = {0: "HMM_SUCCESS", 1: "HMM_ERR_INVALID_VALUE", 2: "HMM_ERR_WORKSPACE", 3: "HMM_ERR_UNSUPPORTED",
          4: "HMM_ERR_CUDA"}


class HmmError(RuntimeError):
    pass


_lib = None


def lib() -> ctypes.CDLL:
    """Loads libhmmscan.so (built in-tree by ``__graft_entry__.build()`` / ``build.py``); fails loudly."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise HmmError(f"{LIB} is missing: build it with `python -m paper_2102_05743_b200.build`")
        L = ctypes.CDLL(LIB)
        i32, i64, p, sz = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t
        L.hmm_status_string.restype = ctypes.c_char_p
        L.hmm_status_string.argtypes = [i32]
        L.hmm_version.restype = ctypes.c_char_p
        L.hmm_workspace_size.restype = sz
        L.hmm_workspace_size.argtypes = [i32, i32, i64, i64]
        L.hmm_smooth.argtypes = [i32, i64, p, p, p, p, p, p, p, p, sz, p]
        L.hmm_viterbi.argtypes = [i32, i64, p, p, p, p, p, p, p, sz, p]
        L.hmm_smooth_batched.argtypes = [i32, i64, i64, p, p, p, p, p, p, p, p, sz, p]
        L.hmm_viterbi_batched.argtypes = [i32, i64, i64, p, p, p, p, p, p, p, sz, p]
        L.hmm_debug_set_timers.argtypes = [p]
        L.hmm_debug_set_timers.restype = None
        L.hmm_debug_plan.argtypes = [i32, i32, i64, i64, p]
        L.hmm_smooth_stats.argtypes = [i32, i64, p, p, p, p, p, p, p, p, p, p, sz, p]
        L.hmm_smooth_stats.restype = i32
        L.hmm_smooth_symbols.argtypes = [i32, i32, i64, p, p, p, p, p, p, p, p, p, sz, p]
        L.hmm_smooth_symbols.restype = i32
        L.hmm_viterbi_symbols.argtypes = [i32, i32, i64, p, p, p, p, p, p, p, p, sz, p]
        L.hmm_viterbi_symbols.restype = i32
        L.hmm_debug_force_path.argtypes = [i32]
        L.hmm_debug_force_path.restype = None
        L.hmm_viterbi_maxproduct.argtypes = [i32, i64, i64, p, p, p, ctypes.c_float, p, p, p, p, p, p, sz, p]
        L.hmm_viterbi_maxproduct.restype = i32
        L.hmm_viterbi_path_elements.argtypes = [i32, i64, i64, p, p, p, p, p, p, p, sz, p]
        L.hmm_viterbi_path_elements.restype = i32
        L.hmm_smooth_varlen.argtypes = [i32, i64, i64, p, p, p, i32, p, p, p, p, p, p, sz, p]
        L.hmm_smooth_varlen.restype = i32
        L.hmm_viterbi_varlen.argtypes = [i32, i64, i64, p, p, p, i32, p, p, p, p, p, sz, p]
        L.hmm_viterbi_varlen.restype = i32
        L.hmm_debug_plan.restype = i32
        for f in ("hmm_smooth", "hmm_viterbi", "hmm_smooth_batched", "hmm_viterbi_batched"):
            getattr(L, f).restype = i32
        _lib = L
    return _lib


def header_symbols() -> list[str]:
    """Function names declared in include/hmmscan.h (the boundary contract)."""
    with open(os.path.join(ROOT, "include", "hmmscan.h")) as f:
        txt = f.read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(hmm_[a-z_0-9]+)\s*\(", txt)))


def plan(op: int, D: int, T: int, B: int = 1) -> dict:
    """Launch plan chosen by the library (introspection)."""
    out = (ctypes.c_int64 * 8)()
    if not lib().hmm_debug_plan(op, D, T, B, out):
        raise HmmError("unsupported shape")
    keys = ["G", "R", "S", "chunk", "K", "fused", "smem", "NT"]
    return dict(zip(keys, list(out)))


def force_path(path: int):
    """Testing/profiling (calling thread only): 0 automatic, 1 lane-streaming, 2 resident/chunked,
    3 large-D leaves on CUDA cores (no tcgen05), 4 batch-parallel plan for 9 <= D <= 32, 5 never it."""
    lib().hmm_debug_force_path(int(path))


def set_timers(buf):
    """Profiling: device int64 buffer [B*G*16] receiving CTA phase timestamps (None disables)."""
    lib().hmm_debug_set_timers(None if buf is None else ctypes.c_void_p(buf.data_ptr()))


def _check(status: int, what: str):
    if status != 0:
        raise HmmError(f"{what}: {STATUS.get(status, status)}")


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


_ws_cache: dict = {}


def workspace_size(op: int, D: int, T: int, B: int = 1) -> int:
    return int(lib().hmm_workspace_size(op, D, T, B))


def workspace(op: int, D: int, T: int, B: int = 1, device=None, stream=None) -> torch.Tensor:
    """Zero-filled device workspace (cached per device/shape/stream; the kernels leave it zeroed).

    Calls that may run concurrently need distinct workspaces (hmmscan.h), so the cache is keyed by the
    stream as well: two streams never share one (the grid-barrier counters would collide)."""
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    sid = None if stream is None else int(stream.cuda_stream)
    key = (device, op, D, T, B, sid)
    ws = _ws_cache.get(key)
    if ws is None:
        n = workspace_size(op, D, T, B)
        if n == 0:
            raise HmmError(f"unsupported shape op={op} D={D} T={T} B={B}")
        ws = torch.zeros(n, dtype=torch.uint8, device=device)
        _ws_cache[key] = ws
    return ws


def _inputs(log_pi, log_A, log_lik):
    if not (log_lik.is_cuda and log_pi.is_cuda and log_A.is_cuda):
        raise HmmError("inputs must be CUDA tensors (no CPU fallback)")
    for t in (log_pi, log_A, log_lik):
        if t.dtype != torch.float32 or not t.is_contiguous():
            raise HmmError("inputs must be contiguous float32")
    batched = log_lik.dim() == 3
    B = log_lik.shape[0] if batched else 1
    T, D = log_lik.shape[-2], log_lik.shape[-1]
    if tuple(log_pi.shape) != (D,) or tuple(log_A.shape) != (D, D):
        raise HmmError("shape mismatch: log_pi [D], log_A [D, D], log_lik [T, D] or [B, T, D]")
    return batched, B, T, D


def smooth(log_pi, log_A, log_lik, want_filtered: bool = True, out=None, ws=None, stream=None):
    """Parallel sum-product smoother (Algorithm 3).

    Returns (filtered or None, smoothed, log_likelihood [B] float64, info [B] int32), all on device.
    """
    batched, B, T, D = _inputs(log_pi, log_A, log_lik)
    dev = log_lik.device
    if out is None:
        filt = torch.empty_like(log_lik) if (want_filtered or D > 8) else None
        sm = torch.empty_like(log_lik)
        lz = torch.empty(B, dtype=torch.float64, device=dev)
        info = torch.empty(B, dtype=torch.int32, device=dev)
    else:
        filt, sm, lz, info = out
    ws = workspace(HMM_OP_SMOOTH, D, T, B, dev, stream) if ws is None else ws
    L = lib()
    if batched:
        st = L.hmm_smooth_batched(D, T, B, _ptr(log_pi), _ptr(log_A), _ptr(log_lik), _ptr(filt), _ptr(sm),
                                  _ptr(lz), _ptr(info), _ptr(ws), ws.numel(), _stream(stream))
    else:
        st = L.hmm_smooth(D, T, _ptr(log_pi), _ptr(log_A), _ptr(log_lik), _ptr(filt), _ptr(sm), _ptr(lz),
                          _ptr(info), _ptr(ws), ws.numel(), _stream(stream))
    _check(st, "hmm_smooth")
    return filt, sm, lz, info


def smooth_stats(log_pi, log_A, log_lik, want_marginals: bool = True, stream=None):
    """Smoother + Baum-Welch E-step statistics for one sequence, 1 <= D <= 8.

    Returns (filtered or None, smoothed or None, log_likelihood [1], xi_sum [D,D] f64, gamma_sum [D] f64,
    info [1]); xi_sum(i,j) = sum_t p(x_{t-1}=i, x_t=j | y), gamma_sum(d) = sum_t p(x_t=d | y).
    """
    batched, B, T, D = _inputs(log_pi, log_A, log_lik)
    if batched:
        raise HmmError("smooth_stats: one sequence")
    dev = log_lik.device
    filt = torch.empty_like(log_lik) if want_marginals else None
    sm = torch.empty_like(log_lik) if want_marginals else None
    lz = torch.empty(1, dtype=torch.float64, device=dev)
    xi = torch.empty((D, D), dtype=torch.float64, device=dev)
    g = torch.empty(D, dtype=torch.float64, device=dev)
    info = torch.empty(1, dtype=torch.int32, device=dev)
    ws = workspace(HMM_OP_SMOOTH_STATS, D, T, 1, dev, stream)
    st = lib().hmm_smooth_stats(D, T, _ptr(log_pi), _ptr(log_A), _ptr(log_lik), _ptr(filt), _ptr(sm), _ptr(lz),
                                _ptr(xi), _ptr(g), _ptr(info), _ptr(ws), ws.numel(), _stream(stream))
    _check(st, "hmm_smooth_stats")
    return filt, sm, lz, xi, g, info


def _sym_inputs(log_pi, log_A, log_B, y):
    for name, t in (("log_pi", log_pi), ("log_A", log_A), ("log_B", log_B), ("y", y)):
        if not t.is_cuda:
            raise HmmError(f"{name} must be a CUDA tensor (no CPU path)")
    if y.dtype != torch.uint8 or y.dim() != 1 or not y.is_contiguous():
        raise HmmError("y: contiguous uint8 [T]")
    for name, t in (("log_pi", log_pi), ("log_A", log_A), ("log_B", log_B)):
        if t.dtype != torch.float32 or not t.is_contiguous():
            raise HmmError(f"{name}: contiguous float32")
    if log_B.dim() != 2:
        raise HmmError("log_B: [D, V]")
    D, V = log_B.shape
    if tuple(log_pi.shape) != (D,) or tuple(log_A.shape) != (D, D):
        raise HmmError("shape mismatch: log_pi [D], log_A [D, D], log_B [D, V]")
    return D, V, y.numel()


def smooth_symbols(log_pi, log_A, log_B, y, want_filtered: bool = True, stream=None):
    """Smoother over discrete observations y [T] uint8 with emissions log_B [D, V].
    Returns (filtered or None, smoothed, log_likelihood [1], info [1])."""
    D, V, T = _sym_inputs(log_pi, log_A, log_B, y)
    dev = y.device
    filt = torch.empty((T, D), dtype=torch.float32, device=dev) if want_filtered else None
    sm = torch.empty((T, D), dtype=torch.float32, device=dev)
    lz = torch.empty(1, dtype=torch.float64, device=dev)
    info = torch.empty(1, dtype=torch.int32, device=dev)
    ws = workspace(HMM_OP_SMOOTH, D, T, 1, dev, stream)
    st = lib().hmm_smooth_symbols(D, V, T, _ptr(log_pi), _ptr(log_A), _ptr(log_B), _ptr(y), _ptr(filt), _ptr(sm),
                                  _ptr(lz), _ptr(info), _ptr(ws), ws.numel(), _stream(stream))
    _check(st, "hmm_smooth_symbols")
    return filt, sm, lz, info


def viterbi_symbols(log_pi, log_A, log_B, y, stream=None):
    """MAP path over discrete observations.  Returns (path [T] int32, log_prob [1], info [1])."""
    D, V, T = _sym_inputs(log_pi, log_A, log_B, y)
    dev = y.device
    path = torch.empty(T, dtype=torch.int32, device=dev)
    lp = torch.empty(1, dtype=torch.float64, device=dev)
    info = torch.empty(1, dtype=torch.int32, device=dev)
    ws = workspace(HMM_OP_VITERBI, D, T, 1, dev, stream)
    st = lib().hmm_viterbi_symbols(D, V, T, _ptr(log_pi), _ptr(log_A), _ptr(log_B), _ptr(y), _ptr(path), _ptr(lp),
                                   _ptr(info), _ptr(ws), ws.numel(), _stream(stream))
    _check(st, "hmm_viterbi_symbols")
    return path, lp, info


def viterbi(log_pi, log_A, log_lik, out=None, ws=None, stream=None):
    """Parallel max-product MAP path (Def. 5 + backpointers).  Returns (path int32, log_prob f64 [B], info [B])."""
    batched, B, T, D = _inputs(log_pi, log_A, log_lik)
    dev = log_lik.device
    if out is None:
        path = torch.empty(log_lik.shape[:-1], dtype=torch.int32, device=dev)
        lp = torch.empty(B, dtype=torch.float64, device=dev)
        info = torch.empty(B, dtype=torch.int32, device=dev)
    else:
        path, lp, info = out
    ws = workspace(HMM_OP_VITERBI, D, T, B, dev, stream) if ws is None else ws
    L = lib()
    if batched:
        st = L.hmm_viterbi_batched(D, T, B, _ptr(log_pi), _ptr(log_A), _ptr(log_lik), _ptr(path), _ptr(lp),
                                   _ptr(info), _ptr(ws), ws.numel(), _stream(stream))
    else:
        st = L.hmm_viterbi(D, T, _ptr(log_pi), _ptr(log_A), _ptr(log_lik), _ptr(path), _ptr(lp), _ptr(info),
                           _ptr(ws), ws.numel(), _stream(stream))
    _check(st, "hmm_viterbi")
    return path, lp, info


def viterbi_maxproduct(log_pi, log_A, log_lik, tie_tol: float = 0.0, stream=None):
    """Algorithm 5: per-step argmax of the max-product forward x backward potentials
    (Eq. 21) with SPEC's coherence diagnostic.  A validation mode; hmm_viterbi is the production path.
    Returns (path, log_prob [B] f64, path_weight [B] f64, n_tied [B] i64, info [B] i32) on device; info is
    HMM_INFO_AMBIGUOUS where the Eq. 21 assembly is not a MAP path."""
    batched, B, T, D = _inputs(log_pi, log_A, log_lik)
    dev = log_lik.device
    path = torch.empty(log_lik.shape[:-1], dtype=torch.int32, device=dev)
    lp = torch.empty(B, dtype=torch.float64, device=dev)
    pw = torch.empty(B, dtype=torch.float64, device=dev)
    nt = torch.empty(B, dtype=torch.int64, device=dev)
    info = torch.empty(B, dtype=torch.int32, device=dev)
    ws = workspace(HMM_OP_VITERBI_MAXPRODUCT, D, T, B, dev, stream)
    st = lib().hmm_viterbi_maxproduct(D, T, B, _ptr(log_pi), _ptr(log_A), _ptr(log_lik), float(tie_tol), _ptr(path),
                                      _ptr(lp), _ptr(pw), _ptr(nt), _ptr(info), _ptr(ws), ws.numel(), _stream(stream))
    _check(st, "hmm_viterbi_maxproduct")
    return path, lp, pw, nt, info


def viterbi_path_elements(log_pi, log_A, log_lik, stream=None):
    """Definition 4 path-element reduction (Corollary 1), T <= 1024.
    Returns (path, log_prob [B] f64, info [B] i32) on device."""
    batched, B, T, D = _inputs(log_pi, log_A, log_lik)
    dev = log_lik.device
    path = torch.empty(log_lik.shape[:-1], dtype=torch.int32, device=dev)
    lp = torch.empty(B, dtype=torch.float64, device=dev)
    info = torch.empty(B, dtype=torch.int32, device=dev)
    ws = workspace(HMM_OP_VITERBI_PATHELEM, D, T, B, dev, stream)
    st = lib().hmm_viterbi_path_elements(D, T, B, _ptr(log_pi), _ptr(log_A), _ptr(log_lik), _ptr(path), _ptr(lp),
                                         _ptr(info), _ptr(ws), ws.numel(), _stream(stream))
    _check(st, "hmm_viterbi_path_elements")
    return path, lp, info


def _varlen_inputs(log_pi, log_A, log_lik, offsets, max_T):
    for t in (log_pi, log_A, log_lik, offsets):
        if not t.is_cuda:
            raise HmmError("inputs must be CUDA tensors (no CPU fallback)")
        if not t.is_contiguous():
            raise HmmError("inputs must be contiguous")
    for t in (log_pi, log_A, log_lik):
        if t.dtype != torch.float32:
            raise HmmError("log_pi, log_A, log_lik must be float32")
    if offsets.dtype != torch.int64 or offsets.dim() != 1 or offsets.numel() < 2:
        raise HmmError("offsets must be a 1-D int64 tensor [B+1]")
    if log_lik.dim() != 2:
        raise HmmError("log_lik must be packed [N, D]")
    B, D = offsets.numel() - 1, log_lik.shape[1]
    per_seq = log_pi.dim() == 2
    if per_seq:
        if tuple(log_pi.shape) != (B, D) or tuple(log_A.shape) != (B, D, D):
            raise HmmError("per-sequence models: log_pi [B, D], log_A [B, D, D]")
    elif tuple(log_pi.shape) != (D,) or tuple(log_A.shape) != (D, D):
        raise HmmError("shared model: log_pi [D], log_A [D, D]")
    if int(max_T) < 1:
        raise HmmError("max_T must be >= 1")
    return B, D, int(per_seq)


def smooth_varlen(log_pi, log_A, log_lik, offsets, max_T: int, stream=None):
    """Variable-length batch smoother: sequence b = rows [offsets[b], offsets[b+1]) of
    the packed log_lik [N, D]; log_pi/log_A shared ([D], [D, D]) or per sequence ([B, D], [B, D, D]).
    Returns (filtered [N, D], smoothed [N, D], log_likelihood [B] f64, info [B] i32) on device."""
    B, D, per_seq = _varlen_inputs(log_pi, log_A, log_lik, offsets, max_T)
    dev = log_lik.device
    filt = torch.empty_like(log_lik)
    sm = torch.empty_like(log_lik)
    lz = torch.empty(B, dtype=torch.float64, device=dev)
    info = torch.empty(B, dtype=torch.int32, device=dev)
    ws = workspace(HMM_OP_SMOOTH_VARLEN, D, int(max_T), B, dev, stream)
    st = lib().hmm_smooth_varlen(D, B, int(max_T), _ptr(offsets), _ptr(log_pi), _ptr(log_A), per_seq, _ptr(log_lik),
                                 _ptr(filt), _ptr(sm), _ptr(lz), _ptr(info), _ptr(ws), ws.numel(), _stream(stream))
    _check(st, "hmm_smooth_varlen")
    return filt, sm, lz, info


def viterbi_varlen(log_pi, log_A, log_lik, offsets, max_T: int, stream=None):
    """Variable-length batch MAP paths (f4).  Returns (path [N] i32, log_prob [B] f64, info [B] i32)."""
    B, D, per_seq = _varlen_inputs(log_pi, log_A, log_lik, offsets, max_T)
    dev = log_lik.device
    path = torch.empty(log_lik.shape[0], dtype=torch.int32, device=dev)
    lp = torch.empty(B, dtype=torch.float64, device=dev)
    info = torch.empty(B, dtype=torch.int32, device=dev)
    ws = workspace(HMM_OP_VITERBI_VARLEN, D, int(max_T), B, dev, stream)
    st = lib().hmm_viterbi_varlen(D, B, int(max_T), _ptr(offsets), _ptr(log_pi), _ptr(log_A), per_seq, _ptr(log_lik),
                                  _ptr(path), _ptr(lp), _ptr(info), _ptr(ws), ws.numel(), _stream(stream))
    _check(st, "hmm_viterbi_varlen")
    return path, lp, info
