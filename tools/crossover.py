"""Resident (fused) vs lane-streaming decomposition across T (GE D=4): which is faster where."""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
import paper_2102_05743_b200 as H
dev = torch.device("cuda")
fw = torch.empty(512 << 18, device=dev)
def timeit(fn, n=20):
    ts = []
    for i in range(n + 3):
        fw.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        if i >= 3: ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)
for T in [100_000, 300_000, 1_000_000, 1_800_000, 3_000_000]:
    wl = W.ge(T, 1)
    lp, la, ll = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (wl.log_pi, wl.log_A, wl.log_lik))
    row = []
    for path in (2, 1):
        H.force_path(path)
        pl = H.plan(0, 4, T)
        row.append((path, pl["fused"], timeit(lambda: H.smooth(lp, la, ll)), timeit(lambda: H.viterbi(lp, la, ll))))
    H.force_path(0)
    print(f"T={T}: " + "; ".join(f"path{p} (kind {k}) smooth {a:.1f} us viterbi {b:.1f} us" for p, k, a, b in row), flush=True)
