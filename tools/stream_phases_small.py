"""Phase stamps of the streaming kernel at a small T (fixed costs), forced path, GE D=4."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
import paper_2102_05743_b200 as H
T = int(float(sys.argv[1])) if len(sys.argv) > 1 else 12_500
H.force_path(1)
dev = torch.device("cuda")
wl = W.ge(T, 5)
lp, la, ll = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (wl.log_pi, wl.log_A, wl.log_lik))
names = ["start", "pass1", "root pub", "barrier", "exchange", "tree_down", "pass2", "map/exch2", "pass3", "pre-final", "end", "w7 pass1", "w7 pass2"]
for op in (0, 1):
    pl = H.plan(op, 4, T); G = pl["G"]
    buf = torch.zeros(G * 16, dtype=torch.int64, device=dev)
    for rep in range(4):
        H.set_timers(buf if rep == 3 else None)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        (H.smooth if op == 0 else H.viterbi)(lp, la, ll)
        e1.record(); torch.cuda.synchronize()
    H.set_timers(None)
    t = buf.view(G, 16).cpu().numpy().astype(np.float64)
    t0 = t[:, 0].min()
    print(f"op={op} plan={pl} event {e0.elapsed_time(e1)*1e3:.1f} us")
    for i, nm in enumerate(names):
        col = t[:, i]
        if (col == 0).all(): continue
        col = (col - t0) / 1e3
        print(f"  {i:2d} {nm:10s} med {np.median(col):8.2f}  max {col.max():8.2f} us")
