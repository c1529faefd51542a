"""Batch-parallel plan (force 4) vs block scan (force 5) for D = 16 / 32, T = 4096: device ms per call
at several B — the data behind the planner's crossover (hmm_abi.cu use_batchseq)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
import paper_2102_05743_b200 as H

dev = torch.device("cuda")


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for D in (16, 32):
    for B in (128, 256, 512, 1024, 2048):
        wl = W.dense_batch(B, D, 4096) if B <= 1024 else W.random_potentials(D, 4096, seed=1, B=B)
        lp, la, ll = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (wl.log_pi, wl.log_A, wl.log_lik))
        row = [f"D={D} B={B:5d}"]
        for force in (4, 5):
            H.force_path(force)
            ts = timed(lambda: H.smooth(lp, la, ll))
            tv = timed(lambda: H.viterbi(lp, la, ll))
            H.force_path(0)
            row.append(f"{'batchseq' if force == 4 else 'scan'}: smooth {ts:.3f} ms viterbi {tv:.3f} ms")
        print("  ".join(row), flush=True)
        del lp, la, ll
