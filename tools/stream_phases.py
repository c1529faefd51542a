"""Per-CTA phase stamps of the lane-streaming kernel (hmm_debug_set_timers), GE D=4."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
import paper_2102_05743_b200 as H
T = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
dev = torch.device("cuda")
wl = W.ge(T, 5)
lp, la, ll = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (wl.log_pi, wl.log_A, wl.log_lik))
flush = torch.empty(512 << 18, device=dev)
names = ["start", "pass1", "root pub", "barrier", "exchange", "tree_down", "pass2", "map/exch2", "pass3", "pre-final", "end", "w7 pass1", "w7 pass2"]
for op in (0, 1):
    pl = H.plan(op, 4, T)
    G = pl["G"]
    buf = torch.zeros(G * 16, dtype=torch.int64, device=dev)
    for rep in range(3):
        flush.zero_()
        H.set_timers(buf if rep == 2 else None)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if op == 0:
            H.smooth(lp, la, ll)
        else:
            H.viterbi(lp, la, ll)
        e1.record(); torch.cuda.synchronize()
    H.set_timers(None)
    print(f"op={op} plan={pl} event {e0.elapsed_time(e1)*1e3:.1f} us")
    t = buf.view(G, 16).cpu().numpy().astype(np.float64)
    t0 = t[:, 0].min()
    for i, nm in enumerate(names):
        col = t[:, i]
        if (col == 0).all():
            continue
        col = (col - t0) / 1e3
        print(f"  {i:2d} {nm:10s} min {col.min():9.1f}  med {np.median(col):9.1f}  max {col.max():9.1f} us")
    if len(sys.argv) > 2 and op == 0:  # per-CTA pass-2 duration with the SM id, sorted
        p2 = (t[:, 6] - t[:, 5]) / 1e3; p1 = (t[:, 1] - t[:, 0]) / 1e3
        for j in np.argsort(p2):
            print(f"    cta {j:3d} sm {int(t[j, 13]):3d}  pass1 {p1[j]:7.1f}  pass2 {p2[j]:7.1f} us")
    for i in (1, 2, 6, 10, 11, 12):
        col = (t[:, i] - t0) / 1e3
        idx = np.argsort(-col)[:4]
        print(f"  slowest at stamp {i}: " + ", ".join(f"cta {j}: {col[j]:.1f}" for j in idx))
