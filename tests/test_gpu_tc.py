"""Tensor-core (tcgen05 TF32x3) leaf products of the large-D sum-product scan (hmm_large_tc.cu).

Accuracy check stated in DESIGN.md §6.3: every operand is split into a TF32 head and an fp32 tail and
three MMAs are accumulated in fp32 (TF32x3).  These tests hold the tensor-core path to the same bars
as the FP32 CUDA-core path it replaces (marginals 1e-5 abs, log Z 1e-6 rel vs the fp64 oracle), check
the two engines agree with each other, and cover ragged leaf pairs, batches, padding (D < 64) and
device-detected errors.
"""
import numpy as np
import pytest
import torch

import oracle
import workloads as W
import paper_2102_05743_b200 as H
from parity import TOL_MARG, TOL_REL, check_smooth, gpu_smooth, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    H.lib()
    yield
    H.force_path(0)


@pytest.mark.parametrize("D,T", [(64, 1), (64, 17), (64, 1000), (64, 33_333), (33, 5000), (40, 12_345), (57, 2049)])
def test_tc_smoother_vs_oracle(D, T):
    wl = W.dense(D, T, seed=D + T)
    check_smooth(wl, *gpu_smooth(wl))


@pytest.mark.parametrize("D,T", [(64, 20_000), (48, 7000)])
def test_tc_matches_cuda_core_engine(D, T):
    wl = W.dense(D, T, seed=7)
    H.force_path(0)
    a = gpu_smooth(wl)
    H.force_path(3)
    b = gpu_smooth(wl)
    H.force_path(0)
    assert float(np.abs(a[1] - b[1]).max()) <= 2 * TOL_MARG
    assert float(np.abs(a[0] - b[0]).max()) <= 2 * TOL_MARG
    assert rel(a[2][0], b[2][0]) <= TOL_REL


def test_tc_random_potentials():
    """Unnormalised general potentials (rows of A not stochastic, log_lik ~ N(0,1))."""
    wl = W.random_potentials(64, 3000, seed=11)
    check_smooth(wl, *gpu_smooth(wl))


@pytest.mark.parametrize("B,D,T", [(3, 64, 2000), (5, 50, 777)])
def test_tc_batched(B, D, T):
    wl = W.dense_batch(B, D, T)
    dev = torch.device("cuda")
    lp, la, ll = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (wl.log_pi, wl.log_A, wl.log_lik))
    f, s, lz, info = H.smooth(lp, la, ll)
    s = s.cpu().numpy(); lz = lz.cpu().numpy()
    for b in range(B):
        o = oracle.smooth(wl.log_pi, wl.log_A, wl.log_lik[b])
        assert int(info[b]) == 0
        assert float(np.abs(s[b] - o["smoothed"]).max()) <= TOL_MARG
        assert rel(lz[b], o["log_z"]) <= TOL_REL


def test_tc_info_codes():
    wl = W.dense(64, 20_000, seed=3)
    wl.log_lik[12_345, :] = -np.inf
    assert int(gpu_smooth(wl)[3][0]) == 12_346
    wl = W.dense(64, 20_000, seed=3)
    wl.log_lik[777, 5] = np.nan
    assert int(gpu_smooth(wl)[3][0]) == -1
