"""Streaming smoother (GE D=4) at T values that fill every lane exactly vs leave e empty lanes (and
optionally one partial lane) at the end of the last warp: the last CTA's warp-7 pass-1 / pass-2 end
stamps against the median warp 7 of the other CTAs (hmm_debug_set_timers)."""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
import paper_2102_05743_b200 as H
dev = torch.device("cuda")
EX = 148 * 256 * 2640
wl = W.ge(EX, 5)
lp, la = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (wl.log_pi, wl.log_A))
llf = torch.from_numpy(np.ascontiguousarray(wl.log_lik)).to(dev)
flush = torch.empty(512 << 18, device=dev)
cases = [(0, 0), (0, 0), (1, 0), (2, 0), (4, 0), (7, 0), (12, 0), (16, 0), (24, 0), (31, 0), (7, 1000), (7, 2639)]
for e, part in cases:
    T = EX - e * 2640 - part
    ll = llf[:T]
    for op in (0,) if len(sys.argv) < 2 else (0, 1):
        pl = H.plan(op, 4, T)
        G = pl["G"]
        buf = torch.zeros(G * 16, dtype=torch.int64, device=dev)
        ts = []
        for rep in range(7):
            flush.zero_()
            H.set_timers(buf if rep == 6 else None)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            (H.smooth if op == 0 else H.viterbi)(lp, la, ll)
            e1.record(); torch.cuda.synchronize()
            if 1 <= rep <= 5: ts.append(e0.elapsed_time(e1) * 1e3)
        H.set_timers(None)
        t = buf.view(G, 16).cpu().numpy().astype(np.float64)
        t = (t - t[:, 0].min()) / 1e3
        print(f"empty={e:2d} partial={part:4d} op={op} event {statistics.median(ts):7.1f} us | w7 pass1 med {np.median(t[:-1,11]):6.1f} "
              f"last {t[G-1,11]:6.1f} | w7 pass2 med {np.median(t[:-1,12]):7.1f} last {t[G-1,12]:7.1f} | end max {t[:,10].max():7.1f}",
              flush=True)
