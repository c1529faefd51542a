"""The boundary used from C (tests/c/abi_smoke.c): compiled against include/hmmscan.h and linked with
libhmmscan.so + cudart only.  CPU: it compiles and links; GPU: it runs and its invariant checks pass."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
LIBDIR = os.path.join(ROOT, "paper_2102_05743_b200", "lib")


def _build(tmp_path):
    exe = str(tmp_path / "abi_smoke")
    cmd = ["gcc", "-std=c99", "-O2", os.path.join(ROOT, "tests", "c", "abi_smoke.c"), "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA, "include"), "-L", LIBDIR, "-L", os.path.join(CUDA, "lib64"), "-lhmmscan",
           "-lcudart", "-lm", "-Wl,-rpath," + LIBDIR, "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_program_compiles_and_links(tmp_path):
    if not os.path.exists(os.path.join(LIBDIR, "libhmmscan.so")):
        pytest.skip("library not built")
    _build(tmp_path)


@pytest.mark.gpu
def test_c_program_runs(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
