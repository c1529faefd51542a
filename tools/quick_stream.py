"""Development check of the lane-streaming kernel: forced path vs the fp64 oracle over D and T."""
import sys, time
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, torch
import workloads as W
import paper_2102_05743_b200 as H
from parity import gpu_smooth, gpu_viterbi, check_smooth, check_viterbi
H.force_path(1)
cases = [(4, 1000), (4, 4099), (4, 100_003), (4, 3_000_000)] + [(D, 20_011) for D in (1, 2, 3, 5, 6, 7, 8)]
for D, T in cases:
    wl = W.ge(T, 1) if D == 4 else W.dense(D, T, 3)
    print("plan", H.plan(0, D, T), flush=True)
    r = gpu_smooth(wl)
    try:
        print(f"smooth D={D} T={T} info {r[3]} err {check_smooth(wl, *r)}", flush=True)
    except AssertionError as e:
        print(f"smooth D={D} T={T} FAIL {e}", flush=True)
    wj = W.ge(T, 1, jitter=0.1) if D == 4 else W.dense(D, T, 3)
    r = gpu_viterbi(wj)
    try:
        print(f"viterbi D={D} T={T} info {r[2]} masked {check_viterbi(wj, *r)}", flush=True)
    except AssertionError as e:
        print(f"viterbi D={D} T={T} FAIL {e}", flush=True)
