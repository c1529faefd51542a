"""Development check of the tensor-core leaf path (D = 33..64 sum-product) vs the oracle and vs the
FP32 CUDA-core path (force_path(3)), with timings."""
import sys, time
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, torch
import workloads as W
import paper_2102_05743_b200 as H
from parity import gpu_smooth, check_smooth, to_dev
for D, T in [(64, 1000), (64, 20_000), (48, 5000), (33, 3000), (64, 100_000)]:
    wl = W.dense(D, T, 3)
    for fp in (0, 3):
        H.force_path(fp)
        r = gpu_smooth(wl)
        try:
            err = check_smooth(wl, *r)
            print(f"D={D} T={T} path={fp} info={r[3]} err={err}", flush=True)
        except AssertionError as e:
            print(f"D={D} T={T} path={fp} FAIL {e}", flush=True)
    H.force_path(0)
wl = W.dense(64, 100_000, 3)
lp, la, ll = to_dev(wl)
for fp in (0, 3):
    H.force_path(fp)
    H.smooth(lp, la, ll); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        H.smooth(lp, la, ll)
    e1.record(); torch.cuda.synchronize()
    print(f"config3 smoother path={fp}: {e0.elapsed_time(e1)/5:.3f} ms", flush=True)
H.force_path(0)
