"""Spread of the per-CTA pass-2 end and kernel end stamps of the streaming smoother (GE D=4)."""
import sys, os, statistics, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
import paper_2102_05743_b200 as H
dev = torch.device("cuda")
T = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
wl = W.ge(T, 5)
lp, la, ll = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (wl.log_pi, wl.log_A, wl.log_lik))
flush = torch.empty(512 << 18, device=dev)
G = H.plan(0, 4, T)["G"]
buf = torch.zeros(G * 16, dtype=torch.int64, device=dev)
for rep in range(40):
    flush.zero_()
    H.set_timers(buf if rep % 10 == 9 else None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); H.smooth(lp, la, ll); e1.record(); torch.cuda.synchronize()
    H.set_timers(None)
    if rep % 10 == 9:
        t = buf.view(G, 16).cpu().numpy().astype(np.float64)
        t = (t - t[:, 0].min()) / 1e3
        q = lambda c: " ".join(f"{x:7.1f}" for x in np.percentile(t[:, c], [0, 50, 90, 99, 100]))
        print(f"rep {rep} event {e0.elapsed_time(e1)*1e3:.1f} | pass2 {q(6)} | w7p2 {q(12)} | end {q(10)} | argmax end {int(np.argmax(t[:,10]))}")
print(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active,power.draw", "--format=csv"], capture_output=True, text=True).stdout)
