"""Seeded synthetic HMM workloads (inputs only — none of the method's arithmetic lives here).

Both the fp64 oracle (``oracle/``) and the CUDA path (``paper_2102_05743_b200``) consume the fp32
arrays produced here, so parity tests compare the two on bit-identical inputs.  The recipes are
described in ``hmmgen.c`` and DESIGN.md §"Input recipe"; the GE model is Eq. 22 of the paper
 with the §VI parameters.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hmmgen.c")
_LIB = os.path.join(_HERE, "libhmmgen.so")

GE_PARAMS = dict(p0=0.03, p1=0.1, p2=0.05, q0=0.01, q1=0.1)


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def _L():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        d, i64, u64, i32 = ctypes.c_double, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int
        p = ctypes.c_void_p
        _lib.hmmgen_uniform.restype = d
        _lib.hmmgen_uniform.argtypes = [u64, u64]
        _lib.hmmgen_normal.restype = d
        _lib.hmmgen_normal.argtypes = [u64, u64]
        _lib.hmmgen_uniform_fill.argtypes = [u64, u64, i64, p]
        _lib.hmmgen_ge_model.argtypes = [d, d, d, d, d, p, p, p]
        _lib.hmmgen_simulate_discrete.argtypes = [i32, i32, p, p, p, i64, u64, p, p]
        _lib.hmmgen_loglik_discrete.argtypes = [i32, i32, p, i64, p, p]
        _lib.hmmgen_dense_model.argtypes = [i32, u64, p, p, p]
        _lib.hmmgen_simulate_gaussian.argtypes = [i32, p, p, i64, u64, p, p]
        _lib.hmmgen_jitter.argtypes = [i32, i64, p, d, u64]
        _lib.hmmgen_normal_fill.argtypes = [i64, p, d, d, u64]
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class Workload:
    """One synthetic HMM problem: fp32 log-domain inputs (+ the simulated states, if any)."""

    log_pi: np.ndarray   # [D] float32
    log_A: np.ndarray    # [D, D] float32, log p(x_t = j | x_{t-1} = i)
    log_lik: np.ndarray  # [T, D] or [B, T, D] float32, log p(y_t | x_t = d)
    states: np.ndarray | None = None
    name: str = ""

    @property
    def D(self) -> int:
        return self.log_pi.shape[0]

    @property
    def T(self) -> int:
        return self.log_lik.shape[-2]


def uniform(seed: int, k0: int, n: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    _L().hmmgen_uniform_fill(seed, k0, n, _ptr(out))
    return out


def ge_model(p0=0.03, p1=0.1, p2=0.05, q0=0.01, q1=0.1):
    """Eq. 22: returns (Pi [4,4], O [4,2], prior [4]) in float64."""
    Pi = np.empty((4, 4)); O = np.empty((4, 2)); pr = np.empty(4)
    _L().hmmgen_ge_model(p0, p1, p2, q0, q1, _ptr(Pi), _ptr(O), _ptr(pr))
    return Pi, O, pr


def simulate_discrete(prior, A, O, T: int, seed: int):
    prior = np.ascontiguousarray(prior, np.float64); A = np.ascontiguousarray(A, np.float64)
    O = np.ascontiguousarray(O, np.float64)
    D, V = O.shape
    states = np.empty(T, np.int32); obs = np.empty(T, np.int32)
    _L().hmmgen_simulate_discrete(D, V, _ptr(prior), _ptr(A), _ptr(O), T, seed, _ptr(states), _ptr(obs))
    return states, obs


def loglik_discrete(O, obs) -> np.ndarray:
    O = np.ascontiguousarray(O, np.float64); obs = np.ascontiguousarray(obs, np.int32)
    D, V = O.shape
    out = np.empty((obs.shape[0], D), np.float32)
    _L().hmmgen_loglik_discrete(D, V, _ptr(O), obs.shape[0], _ptr(obs), _ptr(out))
    return out


def ge(T: int, seed: int, jitter: float = 0.0, jitter_seed: int | None = None, **params) -> Workload:
    """GE channel workload (BASELINE configs ①②⑤); optional N(0, jitter^2) on log_lik (near-tie-free copy)."""
    p = dict(GE_PARAMS); p.update(params)
    Pi, O, pr = ge_model(**p)
    states, obs = simulate_discrete(pr, Pi, O, T, seed)
    ll = loglik_discrete(O, obs)
    if jitter > 0:
        _L().hmmgen_jitter(4, T, _ptr(ll), jitter, 7919 + seed if jitter_seed is None else jitter_seed)
    return Workload(np.log(pr).astype(np.float32), np.log(Pi).astype(np.float32), ll, states,
                    f"ge_T{T}_s{seed}" + (f"_j{jitter}" if jitter else ""))


class SymbolWorkload:
    """Discrete-observation workload: log_pi [D], log_A [D,D], log_B [D,V] (log emission matrix), y [T] uint8."""

    def __init__(self, log_pi, log_A, log_B, y, states=None, name=""):
        self.log_pi, self.log_A, self.log_B, self.y, self.states, self.name = log_pi, log_A, log_B, y, states, name
        self.T, self.D, self.V = y.shape[0], log_B.shape[0], log_B.shape[1]


def ge_symbols(T: int, seed: int, **params) -> SymbolWorkload:
    """The GE channel in its native form: y_t in {0,1} with emission matrix O (Eq. 22);
    same chain / observations as ge(T, seed)."""
    p = dict(GE_PARAMS); p.update(params)
    Pi, O, pr = ge_model(**p)
    states, obs = simulate_discrete(pr, Pi, O, T, seed)
    return SymbolWorkload(np.log(pr).astype(np.float32), np.log(Pi).astype(np.float32),
                          np.log(O).astype(np.float32), obs.astype(np.uint8), states, f"ge_sym_T{T}_s{seed}")


def discrete(D: int, V: int, T: int, seed: int) -> SymbolWorkload:
    """Dense Dirichlet(1) transitions (dense_model) and Dirichlet(1) emission rows over V symbols
    (normalised -log u from counter stream 2^40 + seed), simulated chain and observations."""
    log_pi, log_A = dense_model(D, 1000003 + seed)
    u = uniform((1 << 40) + seed, 0, D * V)
    e = -np.log(np.maximum(u, 1e-300)).reshape(D, V)
    B = e / e.sum(1, keepdims=True)
    states, obs = simulate_discrete(np.exp(log_pi.astype(np.float64)), np.exp(log_A.astype(np.float64)), B, T, seed)
    return SymbolWorkload(log_pi, log_A, np.log(B).astype(np.float32), obs.astype(np.uint8), states,
                          f"discrete_D{D}_V{V}_T{T}_s{seed}")


def dense_model(D: int, seed: int):
    log_pi = np.empty(D, np.float32); log_A = np.empty((D, D), np.float32)
    _L().hmmgen_dense_model(D, seed, _ptr(log_pi), _ptr(log_A), None)
    return log_pi, log_A


def dense(D: int, T: int, seed: int, model_seed: int | None = None) -> Workload:
    """Dense Dirichlet(1) model + Gaussian emissions mu_d = d (BASELINE config ③)."""
    log_pi, log_A = dense_model(D, 1000003 + seed if model_seed is None else model_seed)
    states = np.empty(T, np.int32); ll = np.empty((T, D), np.float32)
    _L().hmmgen_simulate_gaussian(D, _ptr(log_pi), _ptr(log_A), T, seed, _ptr(states), _ptr(ll))
    return Workload(log_pi, log_A, ll, states, f"dense_D{D}_T{T}_s{seed}")


def dense_batch(B: int, D: int, T: int, model_seed: int = 424242, seed0: int = 1000) -> Workload:
    """B sequences sharing one dense model; sequence b uses seed seed0+b (BASELINE config ④)."""
    log_pi, log_A = dense_model(D, model_seed)
    ll = np.empty((B, T, D), np.float32); st = np.empty((B, T), np.int32)
    for b in range(B):
        _L().hmmgen_simulate_gaussian(D, _ptr(log_pi), _ptr(log_A), T, seed0 + b, _ptr(st[b]), _ptr(ll[b]))
    return Workload(log_pi, log_A, ll, st, f"dense_B{B}_D{D}_T{T}")


def random_potentials(D: int, T: int, seed: int, B: int | None = None, sigma: float = 1.0) -> Workload:
    """Unnormalised random potentials: log_pi, log_A, log_lik all i.i.d. N(0, sigma^2) (general inputs)."""
    lp = np.empty(D, np.float32); la = np.empty((D, D), np.float32)
    shape = (T, D) if B is None else (B, T, D)
    ll = np.empty(shape, np.float32)
    _L().hmmgen_normal_fill(D, _ptr(lp), 0.0, sigma, 11 + 7 * seed)
    _L().hmmgen_normal_fill(D * D, _ptr(la), 0.0, sigma, 13 + 7 * seed)
    _L().hmmgen_normal_fill(ll.size, _ptr(ll), 0.0, sigma, 17 + 7 * seed)
    return Workload(lp, la, ll, None, f"randpot_D{D}_T{T}_s{seed}")


def planted(D: int, T: int, seed: int, delta: float | None = None, margin: float = 4.0) -> Workload:
    """Planted-path workload: finite log_A, log_pi from a dense model; log_lik_t(d) = -delta*[d != z_t].

    With delta > 2*range(log_A) + range(log_pi) the MAP path is exactly z (SURVEY.md §8(c) closed form v);
    by default delta = that bound + `margin`, so every max-marginal gap is >= margin.
    z is drawn i.i.d. uniform from counters of stream `seed`.
    """
    log_pi, log_A = dense_model(D, 31337 + seed)
    if delta is None:
        rA = float(log_A.max()) - float(log_A.min())
        rp = float(log_pi.max()) - float(log_pi.min())
        delta = 2.0 * rA + rp + margin
    u = uniform(seed, 0, T)
    z = np.minimum((u * D).astype(np.int32), D - 1)
    ll = np.full((T, D), -delta, np.float32)
    ll[np.arange(T), z] = 0.0
    return Workload(log_pi, log_A, ll, z, f"planted_D{D}_T{T}_s{seed}")
