"""Runs the C++ drop-in mirror test (tests/cpp/test_mirror.cpp): the reference's
own forward_lm driven through parse::gpu::GpuProvider vs RoutingProvider, plus
unit parity of the mirrored functions.  The binary is built against the
reference headers in the build container by __graft_entry__.build()."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(__file__), "cpp", "_bin", "test_mirror")


def test_cpp_mirror_drop_in():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    assert os.path.exists(BIN), "tests/cpp/_bin/test_mirror missing: run __graft_entry__.build() where /root/reference exists"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASSED" in r.stdout
