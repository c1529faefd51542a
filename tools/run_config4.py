"""Config 4 (batched B=1024, D=16, T=4096) smoother + Viterbi, twice each (for ncu launch lists)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
import paper_2102_05743_b200 as H
wl = W.dense_batch(1024, 16, 4096)
dev = torch.device("cuda")
lp, la, ll = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (wl.log_pi, wl.log_A, wl.log_lik))
for _ in range(2):
    H.smooth(lp, la, ll); H.viterbi(lp, la, ll)
torch.cuda.synchronize()
