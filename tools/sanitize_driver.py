"""compute-sanitizer driver: one small call of every kernel family through the C ABI, checked against the
oracle, so `compute-sanitizer --tool {memcheck,racecheck,synccheck}` sees each kernel's protocols
(cp.async.bulk + mbarrier staging, the acquire/release grid barrier, tcgen05/TMEM leaves).

  usage: compute-sanitizer --tool racecheck python tools/sanitize_driver.py [family ...]
  families: small stream chunked large tc stats symbols dist batched
"""
import sys

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2102_05743_b200 as H  # noqa: E402
import workloads as W  # noqa: E402
from parity import check_smooth, check_viterbi, gpu_smooth, gpu_viterbi  # noqa: E402


def run(wl, force=0, vit=True):
    H.force_path(force)
    bs = [None] if wl.log_lik.ndim == 2 else list(range(wl.log_lik.shape[0]))
    try:
        r = gpu_smooth(wl)
        for b in bs:
            check_smooth(wl, *r, b=b)
        if vit:
            v = gpu_viterbi(wl)
            for b in bs:
                check_viterbi(wl, *v, b=b)
    finally:
        H.force_path(0)


FAMILIES = {
    "small": lambda: run(W.ge(1000, 0, jitter=0.1)),                         # hmm_small_kernel (resident)
    "stream": lambda: run(W.ge(20011, 1, jitter=0.1), force=1),              # hmm_stream_kernel
    "chunked": lambda: run(W.ge(200003, 2, jitter=0.1), force=2),            # chunked resident plan
    "large": lambda: (run(W.dense(12, 3001, seed=3)), run(W.dense(20, 3001, seed=3)),
                      run(W.dense(40, 3001, seed=3), force=3)),            # lg_* (CUDA cores, DP 16/32/64)
    "tc": lambda: run(W.dense(64, 3001, seed=3), vit=False),                 # lg_leaf_tc_kernel (tcgen05)
    "batched": lambda: (run(W.dense_batch(8, 16, 513)),                      # batched D=16 (lg_*)
                        run(W.random_potentials(4, 1001, 3, B=6))),          # batched D=4 (small kernel)
}


def stats():
    wl = W.ge(20011, 4)
    lp, la, ll = (torch.from_numpy(x).cuda() for x in (wl.log_pi, wl.log_A, wl.log_lik))
    out = H.smooth_stats(lp, la, ll)
    torch.cuda.synchronize()
    assert int(out[-1].item()) == 0


def symbols():
    wl = W.ge_symbols(20011, 5)
    lp, la, lb = (torch.from_numpy(x).cuda() for x in (wl.log_pi, wl.log_A, wl.log_B))
    y = torch.from_numpy(wl.y).cuda()
    f, s, lz, info = H.smooth_symbols(lp, la, lb, y)
    p, lpr, vinfo = H.viterbi_symbols(lp, la, lb, y)
    torch.cuda.synchronize()
    assert int(info.item()) == 0 and int(vinfo.item()) == 0


def variants():
    wl = W.random_potentials(4, 5001, 3, B=2)
    lp, la, ll = (torch.from_numpy(x).cuda() for x in (wl.log_pi, wl.log_A, wl.log_lik))
    out = H.viterbi_maxproduct(lp, la, ll)
    pe = H.viterbi_path_elements(lp, la, ll[:, :1000].contiguous())
    torch.cuda.synchronize()
    assert int(out[-1].abs().max().item()) == 0 and int(pe[-1].abs().max().item()) == 0


def batchseq():
    """bidirectional batch plan (bs3_smooth warp-specialised, bs2_viterbi), both lane-group widths, an odd
    batch (an idle lane group), varlen groups of different lengths, and the one-warp plan"""
    run(W.dense_batch(5, 16, 700, model_seed=3, seed0=1), force=4)
    run(W.dense_batch(3, 32, 301, model_seed=4, seed0=2), force=4)
    run(W.dense_batch(3, 12, 257, model_seed=5, seed0=3), force=6)
    lengths = [100, 700, 33]
    lls = [W.dense(16, n, seed=i, model_seed=9).log_lik for i, n in enumerate(lengths)]
    wl0 = W.dense(16, 10, seed=0, model_seed=9)
    off = torch.tensor(np.concatenate([[0], np.cumsum(lengths)]), dtype=torch.int64).cuda()
    lp, la = torch.from_numpy(wl0.log_pi).cuda(), torch.from_numpy(wl0.log_A).cuda()
    ll = torch.from_numpy(np.concatenate(lls)).cuda()
    H.force_path(4)
    try:
        f, s, lz, info = H.smooth_varlen(lp, la, ll, off, max(lengths))
        p, lpr, vinfo = H.viterbi_varlen(lp, la, ll, off, max(lengths))
        torch.cuda.synchronize()
    finally:
        H.force_path(0)
    assert int(info.abs().max().item()) == 0 and int(vinfo.abs().max().item()) == 0


FAMILIES["batchseq"] = batchseq
FAMILIES["variants"] = variants
FAMILIES["stats"] = stats
FAMILIES["symbols"] = symbols

if __name__ == "__main__":
    names = sys.argv[1:] or list(FAMILIES)
    for n in names:
        FAMILIES[n]()
        torch.cuda.synchronize()
        print("sanitize-driver ok:", n, flush=True)
