"""Pass-1-only launches (split-phase reduce calls) on GE D=4 for ncu captures.  argv: T"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2102_05743_b200.dist import LibBackend
T = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
dev = torch.device("cuda")
wl = W.ge(T, 5, jitter=0.1)
lp, la, ll = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (wl.log_pi, wl.log_A, wl.log_lik))
be = LibBackend()
be.smooth_reduce(lp, la, ll, 0)
be.viterbi_reduce(lp, la, ll, 0)
torch.cuda.synchronize()
