"""fp64 CPU oracle for the HMM hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may import this package.  The product path (``paper_2102_05743_b200``) never imports it and
shares no code with it.

* ``smooth`` / ``viterbi`` / ``max_marginals`` / ``joint_weight`` — sequential fp64 C implementation of
  Algorithm 1, Algorithm 4 and Lemma 3;
  see ``hmm_oracle.c``.
* ``brute`` — exhaustive enumeration over all D^T state sequences of Eqs. 1-3,
  written independently in numpy; it pins the C oracle on tiny inputs.

Parity status: pinned (tests/test_oracle_pins.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hmm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        # No -ffast-math: IEEE fp64 round-to-nearest (SURVEY.md §8(c) reading 15).
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-D_DEFAULT_SOURCE", "-shared", "-fPIC",
                               "-o", _LIB, _SRC, "-lm", "-lpthread"])
    return _LIB


_lib = None


def _L():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        i32, i64, p = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p
        _lib.oracle_smooth.argtypes = [i32, i64, p, p, p, p, p, p, p, p]
        _lib.oracle_viterbi.argtypes = [i32, i64, p, p, p, p, p, p]
        _lib.oracle_smooth_sampled.argtypes = [i32, i64, p, p, p, p, i64, p, p, p, p]
        _lib.oracle_smooth_stats.argtypes = [i32, i64, p, p, p, p, p, p, p]
        _lib.oracle_max_marginals.argtypes = [i32, i64, p, p, p, p, p]
        _lib.oracle_joint_weight.argtypes = [i32, i64, p, p, p, p]
        _lib.oracle_joint_weight.restype = ctypes.c_double
        _lib.oracle_max_marginal_gap.argtypes = [i32, i64, p, p, p, p]
        _lib.oracle_joint_weight_diff.argtypes = [i32, i64, p, p, p, p, p]
        _lib.oracle_joint_weight_diff.restype = ctypes.c_double
        _lib.oracle_smooth_batched.argtypes = [i32, i64, i64, p, p, p, p, p, p, p, p, i32]
        _lib.oracle_viterbi_batched.argtypes = [i32, i64, i64, p, p, p, p, p, p, i32]
    return _lib


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def smooth(log_pi, log_A, log_lik, want_filtered=True, want_smoothed=True):
    """Returns dict(filtered [T,D] f64, smoothed [T,D] f64, log_z, log_z_bwd, info)."""
    log_pi, log_A, log_lik = _f32(log_pi), _f32(log_A), _f32(log_lik)
    T, D = log_lik.shape
    filt = np.empty((T, D)) if want_filtered else None
    sm = np.empty((T, D)) if want_smoothed else None
    lz = ctypes.c_double(); lzb = ctypes.c_double(); info = ctypes.c_int64()
    _L().oracle_smooth(D, T, _p(log_pi), _p(log_A), _p(log_lik), _p(filt), _p(sm),
                       ctypes.byref(lz), ctypes.byref(lzb), ctypes.byref(info))
    return dict(filtered=filt, smoothed=sm, log_z=lz.value, log_z_bwd=lzb.value, info=info.value)


def smooth_sampled(log_pi, log_A, log_lik, ts):
    """Algorithm 1 keeping only the rows at the sample steps `ts` (O(len(ts)) memory, for full-size
    checks).  Returns dict(ts, filtered [n,D], smoothed [n,D], log_z, info); ts sorted, unique."""
    log_pi, log_A, log_lik = _f32(log_pi), _f32(log_A), _f32(log_lik)
    T, D = log_lik.shape
    ts = np.unique(np.asarray(ts, np.int64))
    assert ts.size == 0 or (ts[0] >= 0 and ts[-1] < T)
    filt = np.empty((ts.size, D)); sm = np.empty((ts.size, D))
    lz = ctypes.c_double(); info = ctypes.c_int64()
    _L().oracle_smooth_sampled(D, T, _p(log_pi), _p(log_A), _p(log_lik), _p(ts), ts.size, _p(filt), _p(sm),
                               ctypes.byref(lz), ctypes.byref(info))
    return dict(ts=ts, filtered=filt, smoothed=sm, log_z=lz.value, info=info.value)


def smooth_stats(log_pi, log_A, log_lik):
    """Baum-Welch E-step statistics: dict(xi_sum [D,D] = sum_{t>=1} p(x_{t-1}=i, x_t=j|y),
    gamma_sum [D] = sum_t p(x_t=d|y), log_z, info)."""
    log_pi, log_A, log_lik = _f32(log_pi), _f32(log_A), _f32(log_lik)
    T, D = log_lik.shape
    xi = np.empty((D, D)); g = np.empty(D)
    lz = ctypes.c_double(); info = ctypes.c_int64()
    _L().oracle_smooth_stats(D, T, _p(log_pi), _p(log_A), _p(log_lik), _p(xi), _p(g), ctypes.byref(lz),
                             ctypes.byref(info))
    return dict(xi_sum=xi, gamma_sum=g, log_z=lz.value, info=info.value)


def symbols_loglik(log_B, y):
    """Eq. 5b with discrete observations: log_lik_t(d) = log p(y_t | x_t = d) = log_B[d, y_t]."""
    log_B = _f32(log_B)
    return np.ascontiguousarray(log_B[:, np.asarray(y, np.int64)].T)


def smooth_symbols(log_pi, log_A, log_B, y, want_filtered=True, want_smoothed=True):
    """The smoother of `smooth` on the emissions gathered from the symbol sequence."""
    return smooth(log_pi, log_A, symbols_loglik(log_B, y), want_filtered, want_smoothed)


def viterbi_symbols(log_pi, log_A, log_B, y):
    return viterbi(log_pi, log_A, symbols_loglik(log_B, y))


def viterbi(log_pi, log_A, log_lik):
    """Returns dict(path [T] int32, log_prob, info)."""
    log_pi, log_A, log_lik = _f32(log_pi), _f32(log_A), _f32(log_lik)
    T, D = log_lik.shape
    path = np.empty(T, np.int32)
    lp = ctypes.c_double(); info = ctypes.c_int64()
    _L().oracle_viterbi(D, T, _p(log_pi), _p(log_A), _p(log_lik), _p(path), ctypes.byref(lp), ctypes.byref(info))
    return dict(path=path, log_prob=lp.value, info=info.value)


def max_marginals(log_pi, log_A, log_lik):
    """Returns (score [T,D] = log psi~f + log psi~b, gap [T] = best - second best)."""
    log_pi, log_A, log_lik = _f32(log_pi), _f32(log_A), _f32(log_lik)
    T, D = log_lik.shape
    score = np.empty((T, D)); gap = np.empty(T)
    _L().oracle_max_marginals(D, T, _p(log_pi), _p(log_A), _p(log_lik), _p(score), _p(gap))
    return score, gap


def max_marginal_gap(log_pi, log_A, log_lik):
    """gap [T] float32 = best - second best max-marginal score at every step (as max_marginals' gap,
    bitwise after rounding to float32) in O(T) memory: usable at T = 1e8."""
    log_pi, log_A, log_lik = _f32(log_pi), _f32(log_A), _f32(log_lik)
    T, D = log_lik.shape
    gap = np.empty(T, np.float32)
    if _L().oracle_max_marginal_gap(D, T, _p(log_pi), _p(log_A), _p(log_lik), _p(gap)) != 0:
        raise MemoryError("oracle_max_marginal_gap")
    return gap


def joint_weight_diff(log_pi, log_A, log_lik, path_a, path_b) -> float:
    """log w(path_a) - log w(path_b) (Eq. 6), summed over the differing terms only."""
    log_pi, log_A, log_lik = _f32(log_pi), _f32(log_A), _f32(log_lik)
    a = np.ascontiguousarray(path_a, np.int32); b = np.ascontiguousarray(path_b, np.int32)
    T, D = log_lik.shape
    return _L().oracle_joint_weight_diff(D, T, _p(log_pi), _p(log_A), _p(log_lik), _p(a), _p(b))


def joint_weight(log_pi, log_A, log_lik, path) -> float:
    log_pi, log_A, log_lik = _f32(log_pi), _f32(log_A), _f32(log_lik)
    path = np.ascontiguousarray(path, np.int32)
    T, D = log_lik.shape
    return _L().oracle_joint_weight(D, T, _p(log_pi), _p(log_A), _p(log_lik), _p(path))


def smooth_batched(log_pi, log_A, log_lik, nthreads=None, want_outputs=True):
    log_pi, log_A, log_lik = _f32(log_pi), _f32(log_A), _f32(log_lik)
    B, T, D = log_lik.shape
    nthreads = nthreads or os.cpu_count() or 1
    filt = np.empty((B, T, D)) if want_outputs else None
    sm = np.empty((B, T, D)) if want_outputs else None
    lz = np.empty(B); lzb = np.empty(B); info = np.empty(B, np.int64)
    _L().oracle_smooth_batched(D, T, B, _p(log_pi), _p(log_A), _p(log_lik), _p(filt), _p(sm), _p(lz),
                               _p(lzb), _p(info), nthreads)
    return dict(filtered=filt, smoothed=sm, log_z=lz, log_z_bwd=lzb, info=info)


def viterbi_batched(log_pi, log_A, log_lik, nthreads=None):
    log_pi, log_A, log_lik = _f32(log_pi), _f32(log_A), _f32(log_lik)
    B, T, D = log_lik.shape
    nthreads = nthreads or os.cpu_count() or 1
    path = np.empty((B, T), np.int32); lp = np.empty(B); info = np.empty(B, np.int64)
    _L().oracle_viterbi_batched(D, T, B, _p(log_pi), _p(log_A), _p(log_lik), _p(path), _p(lp), _p(info), nthreads)
    return dict(path=path, log_prob=lp, info=info)
