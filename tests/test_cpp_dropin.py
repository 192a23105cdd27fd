"""Runs the C++ drop-in test (tests/cpp/test_dropin.cpp, built into
oracle/_ref/test_dropin against the reference headers): reference caller code
switched to mrsim::cuda::reset_batch / step_batch reproduces the reference's
outputs over full horizons for every benchmark config."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "test_dropin")


@pytest.mark.gpu
def test_cpp_dropin():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/test_dropin not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
