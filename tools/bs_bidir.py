"""Bidirectional batch-parallel plan (two warps per sequence; force 4 picks it while B fits one wave) vs
the one-warp plan (force 6), D = 16 / 32, T = 4096: device ms per call and agreement of the outputs."""
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


Ds = [int(x) for x in sys.argv[1:]] or [16, 32]
for D in Ds:
    for B in (128, 512, 1024, 2048):
        wl = W.dense_batch(B, D, 4096) if B <= 1024 else W.random_potentials(D, 4096, seed=1, B=B)
        lp, la, ll = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (wl.log_pi, wl.log_A, wl.log_lik))
        row, res = [f"D={D} B={B:5d}"], {}
        for force in (4, 6):
            H.force_path(force)
            ts = timed(lambda: H.smooth(lp, la, ll))
            tv = timed(lambda: H.viterbi(lp, la, ll))
            res[force] = (H.smooth(lp, la, ll), H.viterbi(lp, la, ll))
            H.force_path(0)
            row.append(f"{'bidir' if force == 4 else 'one-warp'}: smooth {ts:.3f} ms viterbi {tv:.3f} ms")
        (f4, s4, z4, i4), (p4, l4, vi4) = res[4]
        (f6, s6, z6, i6), (p6, l6, vi6) = res[6]
        row.append(f"| d_filt {(f4 - f6).abs().max().item():.1e} d_smooth {(s4 - s6).abs().max().item():.1e} "
                   f"d_logz {(z4 - z6).abs().max().item():.1e} d_logp {(l4 - l6).abs().max().item():.1e} "
                   f"path_diff {(p4 != p6).sum().item()} info {int(i4.abs().sum())}/{int(vi4.abs().sum())}")
        print("  ".join(row), flush=True)
        del lp, la, ll
