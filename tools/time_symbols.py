import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, statistics
import workloads as W
import paper_2102_05743_b200 as H
dev = torch.device("cuda")
fw = torch.empty(512 << 18, device=dev)
def timeit(fn, n=10):
    ts = []
    for i in range(n + 3):
        fw.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        if i >= 3: ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)
T = 100_000_000
ws = W.ge_symbols(T, 5)
lp, la, lb, y = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (ws.log_pi, ws.log_A, ws.log_B, ws.y))
ts = timeit(lambda: H.smooth_symbols(lp, la, lb, y))
tv = timeit(lambda: H.viterbi_symbols(lp, la, lb, y))
print(f"GE symbols T=1e8: smoother {ts:.3f} ms ({T/ts*1e3:.3e} steps/s), viterbi {tv:.3f} ms")
