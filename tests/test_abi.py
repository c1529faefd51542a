"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol include/hmmscan.h
declares, and host-side validation rejects bad arguments before any device work."""
import ctypes

import pytest

import paper_2102_05743_b200 as H


@pytest.fixture(scope="module")
def L():
    return H.lib()


def test_exports_every_header_symbol(L):
    names = H.header_symbols()
    assert {"hmm_smooth", "hmm_viterbi", "hmm_smooth_batched", "hmm_viterbi_batched",
            "hmm_workspace_size", "hmm_status_string", "hmm_version"} <= set(names)
    for n in names:
        assert hasattr(L, n), f"libhmmscan.so does not export {n}"


def test_status_strings(L):
    for code, name in H.STATUS.items():
        assert L.hmm_status_string(code).decode() == name
    assert L.hmm_status_string(99).decode() == "HMM_ERR_UNKNOWN"
    assert b"sm_100a" in L.hmm_version()


def test_invalid_arguments_rejected_on_host(L):
    p = ctypes.c_void_p(256)
    # D < 1, T < 1, B < 1
    assert L.hmm_smooth(0, 10, p, p, p, p, p, p, p, p, 1 << 20, None) == 1
    assert L.hmm_smooth(4, 0, p, p, p, p, p, p, p, p, 1 << 20, None) == 1
    assert L.hmm_viterbi(4, -5, p, p, p, p, p, p, p, 1 << 20, None) == 1
    assert L.hmm_smooth_batched(4, 10, 0, p, p, p, p, p, p, p, p, 1 << 20, None) == 1
    # D beyond this build's range
    assert L.hmm_smooth(H.HMM_MAX_D + 1, 10, p, p, p, p, p, p, p, p, 1 << 20, None) == 3
    # large-D smoother needs the filtered buffer (alpha staging)
    assert L.hmm_smooth(16, 10, p, p, p, None, p, p, p, p, 1 << 20, None) == 3
    # NULL required pointers
    assert L.hmm_smooth(4, 10, None, p, p, p, p, p, p, p, 1 << 20, None) == 1
    assert L.hmm_smooth(4, 10, p, p, p, p, None, p, p, p, 1 << 20, None) == 1   # smoothed NULL
    assert L.hmm_viterbi(4, 10, p, p, p, None, p, p, p, 1 << 20, None) == 1      # path NULL
    # misaligned pointer
    q = ctypes.c_void_p(258)
    assert L.hmm_smooth(4, 10, q, p, p, p, p, p, p, p, 1 << 20, None) == 1


def test_workspace_size_invalid(L):
    assert L.hmm_workspace_size(0, 0, 10, 1) == 0
    assert L.hmm_workspace_size(3, 4, 10, 1) == 0   # no such op
    assert L.hmm_workspace_size(2, 9, 10, 1) == 0   # statistics: D <= 8
    assert L.hmm_workspace_size(2, 4, 10, 2) == 0   # statistics: one sequence
    assert L.hmm_workspace_size(0, 4, 0, 1) == 0


def test_no_cpu_fallback():
    import torch
    x = torch.zeros(10, 4)
    with pytest.raises(H.HmmError):
        H.smooth(torch.zeros(4), torch.zeros(4, 4), x)
    with pytest.raises(H.HmmError):
        H.viterbi(torch.zeros(4), torch.zeros(4, 4), x)
