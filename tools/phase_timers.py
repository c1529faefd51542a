"""Per-CTA phase timing of the small-D kernels (GE D=4 T=1e6 by default) via hmm_debug_set_timers."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
import paper_2102_05743_b200 as H

T = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
wl = W.ge(T, 1)
dev = torch.device("cuda")
lp, la, ll = (torch.from_numpy(x).to(dev) for x in (wl.log_pi, wl.log_A, wl.log_lik))
flush = torch.empty(512 << 18, device=dev)
flush_r = torch.ones(256 << 18, device=dev)
names = {0: ["start", "leaf+tree_up", "root published", "barrier released", "exchange done", "tree_down done",
             "alpha done", "beta done", "stores done", "pre-final", "end", "w0 tile landed", "w0 leaf done", "all leaves done"],
         1: ["start", "leaf+tree_up", "root published", "barrier released", "exchange done", "sweep done",
             "ends resolved", "-", "-", "pre-final", "end", "w0 tile landed", "w0 leaf done", "all leaves done"]}
for op in (0, 1):
    pl = H.plan(op, 4, T)
    G = pl["G"]
    buf = torch.zeros(G * 16, dtype=torch.int64, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for it in range(6):
        flush.zero_(); flush_r.sum()
        if it == 5:
            H.set_timers(buf)
            e0.record()
        if op == 0:
            H.smooth(lp, la, ll)
        else:
            H.viterbi(lp, la, ll)
        if it == 5:
            e1.record()
        H.set_timers(None)
    torch.cuda.synchronize()
    print(f"op={op} event time {e0.elapsed_time(e1)*1e3:.2f} us")
    t = buf.view(G, 16).cpu().numpy().astype(np.float64)
    t0 = t[:, 0].min()
    if op == 0:
        cyc = (t[:, 15] - t[:, 14]); ns = (t[:, 6] - t[:, 5])
        print(f"  alpha sweep: median {np.median(cyc):.0f} SM cycles for S={pl['S']} steps "
              f"({np.median(cyc)/pl['S']:.0f} cycles/step); globaltimer {np.median(ns):.0f} ns "
              f"-> {np.median(cyc)/max(np.median(ns),1):.2f} GHz")
    print(f"op={op} plan={pl}")
    for i, nm in enumerate(names[op]):
        col = t[:, i]
        if (col == 0).all() or nm == "-":
            continue
        c = (col - t0) / 1e3
        print(f"  {i:2d} {nm:18s} min {c.min():7.2f} med {np.median(c):7.2f} max {c.max():7.2f} us")
