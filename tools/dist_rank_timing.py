"""Per-rank device time of the split-phase path at W ranks (emulated on one GPU): what one GPU of an
N-GPU run of config 5 spends per step (kernels only; the all-gathers are NCCL's)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2102_05743_b200.dist import LibBackend, partition
dev = torch.device("cuda")
T = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
wl = W.ge(T, 5)
lp, la = torch.from_numpy(wl.log_pi).to(dev), torch.from_numpy(wl.log_A).to(dev)
flush = torch.empty(512 << 18, device=dev)
def ev():
    return torch.cuda.Event(enable_timing=True)
for world in (1, 2, 4, 8):
    sl = [partition(T, world, r) for r in range(world)]
    t0, n = sl[world - 1]
    bes = [LibBackend() for _ in range(world)]
    ll = torch.from_numpy(np.ascontiguousarray(wl.log_lik[t0:t0 + n])).to(dev)
    r = world - 1
    # rank aggregates of all ranks (correct inputs for the finish phases)
    lls = [torch.from_numpy(np.ascontiguousarray(wl.log_lik[a:a + m])).to(dev) for a, m in sl]
    aggs = [bes[q].smooth_reduce(lp, la, lls[q], sl[q][0])[0] for q in range(world)]
    vaggs = [bes[q].viterbi_reduce(lp, la, lls[q], sl[q][0])[0] for q in range(world)]
    agg_all, vagg_all = torch.cat(aggs), torch.cat(vaggs)
    recs = [bes[q].viterbi_forward(lp, la, lls[q], sl[q][0], vagg_all, q, world)[0] for q in range(world)]
    rec_all = torch.cat(recs)
    del lls
    times = {}
    for rep in range(4):
        flush.zero_()
        e = [ev() for _ in range(6)]
        e[0].record(); bes[r].smooth_reduce(lp, la, ll, t0)
        e[1].record(); bes[r].smooth_finish(lp, la, ll, t0, agg_all, r, world)
        e[2].record(); bes[r].viterbi_reduce(lp, la, ll, t0)
        e[3].record(); bes[r].viterbi_forward(lp, la, ll, t0, vagg_all, r, world)
        e[4].record(); bes[r].viterbi_finish(lp, la, ll, t0, rec_all, r, world)
        e[5].record(); torch.cuda.synchronize()
        if rep > 0:
            for k, nm in enumerate(["s_reduce", "s_finish", "v_reduce", "v_forward", "v_finish"]):
                times.setdefault(nm, []).append(e[k].elapsed_time(e[k + 1]) * 1e3)
    tot = sum(min(v) for v in times.values())
    print(f"W={world} T_local={n}: " + ", ".join(f"{k} {min(v):.0f}" for k, v in times.items()) + f" us; total {tot:.0f} us "
          f"-> {T / (tot * 1e-6):.3e} steps/s if every rank matches", flush=True)
