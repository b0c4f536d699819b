"""Runs the C++ drop-in shim test (include/vsprefill_gpu.hpp): reference test bodies
re-pointed from vsp:: to vsp::gpu::, compared with the reference compiled into the same
binary (tests/cpp/shim_test.cpp, built by tests/cpp/Makefile where the headers exist)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(__file__), "cpp", "_build", "shim_test")


def test_cpp_shim_reference_bodies():
    if not os.path.exists(BIN):
        pytest.skip("shim_test not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout.replace("OK: 0 failure", "")
