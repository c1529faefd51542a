"""Config 3 (dense D=64, T=1e5) smoother + Viterbi once each (for ncu launch lists)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
import paper_2102_05743_b200 as H
wl = W.dense(64, 100_000, 3)
dev = torch.device("cuda")
lp, la, ll = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (wl.log_pi, wl.log_A, wl.log_lik))
for _ in range(2):
    H.smooth(lp, la, ll); H.viterbi(lp, la, ll)
torch.cuda.synchronize()
