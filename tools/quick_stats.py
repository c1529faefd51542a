import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, torch
import workloads as W, oracle
import paper_2102_05743_b200 as H
from parity import to_dev
for D, T in [(4, 1000), (4, 100_003), (4, 2_000_003), (1, 5000), (2, 20_011), (3, 20_011), (5, 20_011), (8, 300_001)]:
    wl = W.ge(T, 3) if D == 4 else W.dense(D, T, 3)
    lp, la, ll = to_dev(wl)
    f, s, lz, xi, g, info = H.smooth_stats(lp, la, ll)
    torch.cuda.synchronize()
    o = oracle.smooth_stats(wl.log_pi, wl.log_A, wl.log_lik)
    om = oracle.smooth(wl.log_pi, wl.log_A, wl.log_lik)
    xi, g = xi.cpu().numpy(), g.cpu().numpy()
    dx = np.abs(xi - o["xi_sum"]); dg = np.abs(g - o["gamma_sum"])
    print(f"D={D} T={T} info={int(info[0])} xi abs {dx.max():.3e} rel {(dx / np.maximum(np.abs(o['xi_sum']), 1)).max():.3e} "
          f"gamma abs {dg.max():.3e} rel {(dg/np.maximum(o['gamma_sum'],1)).max():.3e} sm {np.abs(s.cpu().numpy()-om['smoothed']).max():.2e} "
          f"lz rel {abs(float(lz[0])-o['log_z'])/abs(o['log_z']):.2e}", flush=True)
