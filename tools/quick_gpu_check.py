"""Quick GPU sanity run (used during development): GE T=1e3 and 1e6, smoother + Viterbi vs oracle."""
import sys, time
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, torch
import workloads as W
from parity import gpu_smooth, gpu_viterbi, check_smooth, check_viterbi
for T in [1000, 1_000_000, 3_000_000]:
    wl = W.ge(T, 1)
    t0 = time.time(); r = gpu_smooth(wl); print("smooth", T, "info", r[3], time.time() - t0, flush=True)
    try:
        print("  err", check_smooth(wl, *r), flush=True)
    except AssertionError as e:
        print("  FAIL", e, flush=True)
    wj = W.ge(T, 1, jitter=0.1)
    r = gpu_viterbi(wj); print("viterbi", T, "info", r[2], flush=True)
    try:
        print("  masked", check_viterbi(wj, *r), flush=True)
    except AssertionError as e:
        print("  FAIL", e, flush=True)
