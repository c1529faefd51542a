"""Shared comparison helpers for the GPU parity tests (CUDA path vs the fp64 oracle).

Tolerances (BASELINE.json north_star): marginals max-abs <= 1e-5; log-likelihood and Viterbi
log-probability relative <= 1e-6; Viterbi path bit-exact where the oracle's max-marginal gap is
>= TAU (near-tie-free positions); where the MAP is not unique the returned path must still attain
the MAP joint log-probability (several MAP paths are correct, reading 5).
"""
from __future__ import annotations

import json
import os

import numpy as np
import torch

import oracle
import paper_2102_05743_b200 as H

TOL_MARG = 1e-5
TOL_REL = 1e-6
TAU = 1e-3


def record(name: str, **values):
    """Appends one JSON line of measured errors to $HMM_PARITY_LOG (if set): the numbers DESIGN.md quotes."""
    path = os.environ.get("HMM_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps({"test": name, **{k: (float(v) if isinstance(v, (np.floating, float)) else v)
                                                 for k, v in values.items()}}) + "\n")


def to_dev(wl):
    dev = torch.device("cuda")
    return (torch.from_numpy(np.ascontiguousarray(wl.log_pi)).to(dev),
            torch.from_numpy(np.ascontiguousarray(wl.log_A)).to(dev),
            torch.from_numpy(np.ascontiguousarray(wl.log_lik)).to(dev))


def gpu_smooth(wl, want_filtered=True):
    lp, la, ll = to_dev(wl)
    f, s, lz, info = H.smooth(lp, la, ll, want_filtered=want_filtered)
    torch.cuda.synchronize()
    return (None if f is None else f.cpu().numpy(), s.cpu().numpy(), lz.cpu().numpy(), info.cpu().numpy())


def gpu_viterbi(wl):
    lp, la, ll = to_dev(wl)
    path, lpr, info = H.viterbi(lp, la, ll)
    torch.cuda.synchronize()
    return path.cpu().numpy(), lpr.cpu().numpy(), info.cpu().numpy()


def rel(a, b):
    return abs(a - b) / max(1.0, abs(b))


def check_smooth(wl, filt, sm, lz, info, b=None):
    """Compare one sequence (index b of a batch, or the single sequence) against the oracle."""
    ll = wl.log_lik if b is None else wl.log_lik[b]
    o = oracle.smooth(wl.log_pi, wl.log_A, ll)
    assert o["info"] == 0
    i = 0 if b is None else b
    assert int(info[i]) == 0, f"info={info[i]}"
    s = sm if b is None else sm[b]
    err_s = float(np.max(np.abs(s - o["smoothed"])))
    assert err_s <= TOL_MARG, f"smoothed max-abs err {err_s}"
    if filt is not None:
        f = filt if b is None else filt[b]
        err_f = float(np.max(np.abs(f - o["filtered"])))
        assert err_f <= TOL_MARG, f"filtered max-abs err {err_f}"
    r = rel(float(lz[i]), o["log_z"])
    assert r <= TOL_REL, f"log Z rel err {r} ({lz[i]} vs {o['log_z']})"
    return err_s, r


def check_viterbi(wl, path, lpr, info, b=None, strict=None):
    """Bit-exact path where the oracle gap >= TAU; joint log-prob of the GPU path == MAP everywhere."""
    ll = wl.log_lik if b is None else wl.log_lik[b]
    o = oracle.viterbi(wl.log_pi, wl.log_A, ll)
    assert o["info"] == 0
    i = 0 if b is None else b
    assert int(info[i]) == 0, f"info={info[i]}"
    p = path if b is None else path[b]
    r = rel(float(lpr[i]), o["log_prob"])
    assert r <= TOL_REL, f"log_prob rel err {r}"
    _, gap = oracle.max_marginals(wl.log_pi, wl.log_A, ll)
    safe = gap >= TAU
    mism = np.nonzero((p != o["path"]) & safe)[0]
    assert mism.size == 0, f"{mism.size} path mismatches at near-tie-free positions, first {mism[:5]}"
    if strict is True:
        assert safe.all(), "input not near-tie-free"
        assert np.array_equal(p, o["path"])
    jw = oracle.joint_weight(wl.log_pi, wl.log_A, ll, p)
    assert rel(jw, o["log_prob"]) <= TOL_REL, f"GPU path joint log-prob {jw} vs MAP {o['log_prob']}"
    return int((~safe).sum())
