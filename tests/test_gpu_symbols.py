"""GPU parity of the symbol-input entry points: discrete observations y [T] uint8
and emissions log_B [D, V]; the kernels gather log_lik_t = log_B[:, y_t] on chip (1 byte per step of
input instead of 4D).  Compared with the fp64 oracle on the gathered log_lik, and with the log_lik
entry points on the same data."""
import numpy as np
import pytest
import torch

import oracle
import workloads as W
import paper_2102_05743_b200 as H
from parity import TAU, TOL_MARG, TOL_REL, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    H.lib()


def _dev(ws):
    d = torch.device("cuda")
    return tuple(torch.from_numpy(np.ascontiguousarray(x)).to(d) for x in (ws.log_pi, ws.log_A, ws.log_B, ws.y))


def _check(ws, tol_path=True):
    lp, la, lb, y = _dev(ws)
    f, s, lz, info = H.smooth_symbols(lp, la, lb, y)
    path, lpr, vinfo = H.viterbi_symbols(lp, la, lb, y)
    torch.cuda.synchronize()
    o = oracle.smooth_symbols(ws.log_pi, ws.log_A, ws.log_B, ws.y)
    v = oracle.viterbi_symbols(ws.log_pi, ws.log_A, ws.log_B, ws.y)
    assert int(info[0]) == 0 and int(vinfo[0]) == 0
    assert float(np.abs(s.cpu().numpy() - o["smoothed"]).max()) <= TOL_MARG
    assert float(np.abs(f.cpu().numpy() - o["filtered"]).max()) <= TOL_MARG
    assert rel(float(lz[0]), o["log_z"]) <= TOL_REL
    assert rel(float(lpr[0]), v["log_prob"]) <= TOL_REL
    ll = oracle.symbols_loglik(ws.log_B, ws.y)
    p = path.cpu().numpy()
    assert rel(oracle.joint_weight(ws.log_pi, ws.log_A, ll, p), v["log_prob"]) <= TOL_REL
    if tol_path and ws.T <= 300_000:
        _, gap = oracle.max_marginals(ws.log_pi, ws.log_A, ll)
        assert int(((p != v["path"]) & (gap >= TAU)).sum()) == 0


@pytest.mark.parametrize("T", [1, 5, 4099, 100_003, 3_000_001])
def test_ge_symbols(T):
    _check(W.ge_symbols(T, 7))


@pytest.mark.parametrize("D,V", [(1, 3), (2, 2), (3, 5), (5, 17), (6, 64), (7, 200), (8, 256)])
def test_discrete_every_D(D, V):
    _check(W.discrete(D, V, 50_001, seed=D))


def test_symbols_match_loglik_path():
    """Same data through both entry points: identical decompositions, so the outputs agree closely."""
    ws = W.ge_symbols(2_000_000, 4)
    wl = W.ge(2_000_000, 4)
    lp, la, lb, y = _dev(ws)
    ll = torch.from_numpy(wl.log_lik).cuda()
    a = H.smooth_symbols(lp, la, lb, y)
    H.force_path(1)
    b = H.smooth(lp, la, ll)
    H.force_path(0)
    assert float((a[1] - b[1]).abs().max()) <= 1e-6
    assert rel(float(a[2][0]), float(b[2][0])) <= 1e-9


def test_symbol_out_of_range_and_nan():
    ws = W.ge_symbols(10_000, 2)
    ws.y[1234] = 7  # V = 2
    lp, la, lb, y = _dev(ws)
    assert int(H.smooth_symbols(lp, la, lb, y)[3][0]) == -1
    assert int(H.viterbi_symbols(lp, la, lb, y)[2][0]) == -1
    ws = W.ge_symbols(10_000, 2)
    ws.log_B[1, 0] = np.nan
    lp, la, lb, y = _dev(ws)
    assert int(H.smooth_symbols(lp, la, lb, y)[3][0]) == -1
