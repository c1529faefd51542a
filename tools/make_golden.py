#!/usr/bin/env python
"""Regenerates the worked-example fixtures under tests/golden/ from brute-force enumeration.

Only ``oracle/brute.py`` (Eqs. 1-3 of the paper written out over all D^T state sequences, PAPER.md:76-90,
467-471) computes anything here; no value comes from the CUDA path or from the recursive oracle.  The
models are the printed ones:

* ``ge_T5.json``   — the GE channel of Eq. 22 at the §VI parameters (the matrices
                     of ``ge_model.json``), y = [0,1,1,0,0].
* ``spec_D2_T4.json`` — SPEC.md's D=2 model, y = [0,1,1,0].

Inputs are the fp64 logs of the printed probabilities, so the values are the exact-model ones (the tests
compare the fp32-input oracle against them with a 2e-7 allowance for input rounding).

    python tools/make_golden.py           # check: the committed fixtures equal a fresh enumeration
    python tools/make_golden.py --write   # rewrite the computed fields of both fixtures
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import brute  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
TOL = 5e-10  # the fixtures' tol_values: SURVEY printed 10 decimals


def _load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def _fields(lp, la, ll):
    s = brute.smooth(lp, la, ll)
    v = brute.viterbi(lp, la, ll)
    return {"log_z": float(s["log_z"]), "smoothed": s["smoothed"].tolist(), "filtered": s["filtered"].tolist(),
            "map_path": v["path"].tolist(), "map_log_prob": float(v["log_prob"]), "map_gap": float(v["gap"])}


def compute():
    gm = _load("ge_model.json")
    ge = _load("ge_T5.json")
    O = np.array(gm["O"])
    ge_f = _fields(np.log(np.array(gm["prior"])), np.log(np.array(gm["Pi"])), np.log(O[:, ge["obs"]].T))
    sp = _load("spec_D2_T4.json")
    B = np.array(sp["B"])
    lp, la = np.log(np.array(sp["prior"])), np.log(np.array(sp["A"]))
    sp_f = _fields(lp, la, np.log(B[:, sp["obs"]].T))
    # joint weight of states (0,1) for observations (0,1) — Eq. 6 by brute.joint_log_weights
    ll2 = np.log(B[:, [0, 1]].T)
    sp_f["joint_weight_obs01_states01"] = float(brute.joint_log_weights(lp, la, ll2, np.array([[0, 1]]))[0])
    return {"ge_T5.json": ge_f, "spec_D2_T4.json": sp_f}


def _close(a, b, tol):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return a.shape == b.shape and bool(np.all(np.abs(a - b) <= tol))


def check(fresh) -> list[str]:
    bad = []
    for name, fields in fresh.items():
        g = _load(name)
        for k, v in fields.items():
            tol = 1e-4 if k == "map_gap" else TOL  # SURVEY printed the gaps to 4 digits
            if k == "map_path":
                ok = list(g[k]) == list(v)
            else:
                ok = _close(g[k], v, tol)
            if not ok:
                bad.append(f"{name}:{k}: committed {g[k]} vs enumeration {v}")
    return bad


def write(fresh):
    for name, fields in fresh.items():
        g = _load(name)
        g.update(fields)
        g["_generated_by"] = "tools/make_golden.py (oracle/brute.py enumeration over all D^T sequences)"
        with open(os.path.join(GOLDEN, name), "w") as f:
            json.dump(g, f, indent=1)
            f.write("\n")


def main():
    fresh = compute()
    if "--write" in sys.argv:
        write(fresh)
        print("wrote", ", ".join(fresh))
        return
    bad = check(fresh)
    if bad:
        print("\n".join(bad))
        sys.exit(1)
    print("fixtures match the enumeration")


if __name__ == "__main__":
    main()
