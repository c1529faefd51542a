import sys, time
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, torch
import workloads as W
from parity import gpu_smooth, gpu_viterbi, check_smooth, check_viterbi
for D, T in [(16, 2000), (64, 3000), (33, 1000)]:
    wl = W.dense(D, T, 5)
    r = gpu_smooth(wl); print("smooth", D, T, "info", r[3], flush=True)
    try: print("  err", check_smooth(wl, *r), flush=True)
    except AssertionError as e: print("  FAIL", e, flush=True)
    r = gpu_viterbi(wl); print("viterbi", D, T, "info", r[2], flush=True)
    try: print("  masked", check_viterbi(wl, *r), flush=True)
    except AssertionError as e: print("  FAIL", e, flush=True)
