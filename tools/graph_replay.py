"""Eager calls vs CUDA-graph replay of hmm_smooth / hmm_viterbi at small T (launch-latency bound):
device time per call (CUDA events around 50 back-to-back calls, L2 not flushed)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
import paper_2102_05743_b200 as H

dev = torch.device("cuda")
for T in (1000, 100_000, 1_000_000):
    wl = W.ge(T, 1)
    lp, la, ll = (torch.from_numpy(x).to(dev) for x in (wl.log_pi, wl.log_A, wl.log_lik))
    out_s = (torch.empty_like(ll), torch.empty_like(ll), torch.empty(1, dtype=torch.float64, device=dev),
             torch.empty(1, dtype=torch.int32, device=dev))
    out_v = (torch.empty(T, dtype=torch.int32, device=dev), torch.empty(1, dtype=torch.float64, device=dev),
             torch.empty(1, dtype=torch.int32, device=dev))
    s = torch.cuda.Stream()
    ws_s = H.workspace(H.HMM_OP_SMOOTH, 4, T, 1, dev, s)
    ws_v = H.workspace(H.HMM_OP_VITERBI, 4, T, 1, dev, s)
    step = lambda: (H.smooth(lp, la, ll, out=out_s, ws=ws_s, stream=s), H.viterbi(lp, la, ll, out=out_v, ws=ws_v, stream=s))
    with torch.cuda.stream(s):
        for _ in range(3):
            step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(50):
            step()
        e1.record(s)
    torch.cuda.synchronize()
    eager = e0.elapsed_time(e1) / 50 * 1e3
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        g.replay()
        e0.record(s)
        for _ in range(50):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) / 50 * 1e3
    ok = int(out_s[3].item()) == 0 and int(out_v[2].item()) == 0
    print(f"T={T:>8}: smoother+viterbi eager {eager:7.1f} us  graph replay {graph:7.1f} us  info ok {ok}", flush=True)
