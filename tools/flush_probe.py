"""Config-5 smoother device time after different L2 flushes (none / 512 MiB write / write + 256 MiB read /
with a 2 ms idle gap): the clean-L2 flush of bench.py costs nothing measurable, an idle GPU before the
launch costs ~20-30 us (clock ramp).  `profiles/r2/flush_probe.txt`."""
import sys, os, statistics
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import workloads as W
import paper_2102_05743_b200 as H
dev = torch.device("cuda")
wl = W.ge(100_000_000, 5)
ll = torch.from_numpy(np.ascontiguousarray(wl.log_lik)).to(dev)
lp, la = torch.from_numpy(wl.log_pi).to(dev), torch.from_numpy(wl.log_A).to(dev)
T, D = 100_000_000, 4
out_s = (torch.empty(T, D, device=dev), torch.empty(T, D, device=dev), torch.empty(1, dtype=torch.float64, device=dev), torch.empty(1, dtype=torch.int32, device=dev))
ws_s = H.workspace(H.HMM_OP_SMOOTH, D, T, 1, dev)
fw = torch.empty(128 << 20, device=dev); fr = torch.ones(64 << 20, device=dev); acc = torch.zeros((), device=dev)
def f_none(): pass
def f_zero(): fw.zero_()
def f_zero_sum(): fw.zero_(); acc.copy_(fr.sum())
def f_zero_sleep(): fw.zero_(); torch.cuda._sleep(2000000)
def f_zero_sum_sleep(): fw.zero_(); acc.copy_(fr.sum()); torch.cuda._sleep(2000000)
for name, fl in [("none", f_none), ("zero", f_zero), ("zero+sum", f_zero_sum), ("zero+sleep", f_zero_sleep), ("zero+sum+sleep", f_zero_sum_sleep)] * 2:
    ts = []
    for i in range(13):
        fl()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); H.smooth(lp, la, ll, out=out_s, ws=ws_s); e1.record(); torch.cuda.synchronize()
        if i >= 3: ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"{name:16s} med {statistics.median(ts):.1f} min {min(ts):.1f} us", flush=True)
