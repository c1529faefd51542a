"""Device time of each BASELINE config (CUDA events, L2 flushed before each call, median of N)."""
import sys, os, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
import paper_2102_05743_b200 as H
dev = torch.device("cuda")
fw = torch.empty(512 << 18, device=dev); fr = torch.ones(256 << 18, device=dev)
def timeit(fn, n=10):
    ts = []
    for i in range(n + 3):
        fw.zero_(); fr.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        if i >= 3: ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)
res = {}
cfgs = {"1_ge_T1e3": W.ge(1000, 0), "2_ge_T1e6": W.ge(1_000_000, 1), "3_dense_D64_T1e5": W.dense(64, 100_000, 3),
        "4_batch_B1024_D16_T4096": W.dense_batch(1024, 16, 4096)}
if len(sys.argv) > 1 and sys.argv[1] == "big":
    cfgs["ge_T1e7"] = W.ge(10_000_000, 5)
    cfgs["5_ge_T1e8_W1"] = W.ge(100_000_000, 5)
for name, wl in cfgs.items():
    lp, la, ll = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (wl.log_pi, wl.log_A, wl.log_lik))
    steps = ll.numel() // ll.shape[-1]
    ts = timeit(lambda: H.smooth(lp, la, ll))
    tv = timeit(lambda: H.viterbi(lp, la, ll))
    res[name] = dict(steps=steps, smooth_ms=ts, viterbi_ms=tv, smooth_steps_per_s=steps / ts * 1e3,
                     viterbi_steps_per_s=steps / tv * 1e3)
    print(name, json.dumps(res[name]), flush=True)
