"""Quick config-5 timing for kernel iteration: median device time (CUDA events, L2 flushed) of the
smoother and Viterbi at T=1e8 and at a T that fills every lane exactly (no ragged warp)."""
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
    return statistics.median(ts), min(ts)
wl = W.ge(100_000_000, 5)
for T in [int(x) for x in (sys.argv[1:] or [100_000_000, 148 * 256 * 2624])]:
    ll = torch.from_numpy(np.ascontiguousarray(wl.log_lik[:T])).to(dev)
    lp, la = torch.from_numpy(wl.log_pi).to(dev), torch.from_numpy(wl.log_A).to(dev)
    s = timeit(lambda: H.smooth(lp, la, ll)); v = timeit(lambda: H.viterbi(lp, la, ll))
    print(f"T={T}: smoother med {s[0]:.1f} min {s[1]:.1f} us ({48 * T / s[0] / 1e3:.0f} GB/s alg); "
          f"viterbi med {v[0]:.1f} min {v[1]:.1f} us", flush=True)
    del ll
