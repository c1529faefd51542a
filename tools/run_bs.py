"""One batched smoother + Viterbi call on the batch-parallel plan (ncu captures): argv B D T."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
import paper_2102_05743_b200 as H
B, D, T = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (1024, 16, 4096)))
wl = W.dense_batch(B, D, T)
dev = torch.device("cuda")
lp, la, ll = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (wl.log_pi, wl.log_A, wl.log_lik))
H.force_path(4)
H.smooth(lp, la, ll); H.viterbi(lp, la, ll)
torch.cuda.synchronize()
