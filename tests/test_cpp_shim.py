"""The reference's own C++ API driving libskb200 through include/streamk_b200.hpp
(tests/cpp/shim_test.cpp, built against the reference headers/sources by
tests/cpp/Makefile)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "shim_test")


def _binary():
    if not os.path.exists(BIN) and os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    if not os.path.exists(BIN):
        pytest.skip("shim_test not built (needs the reference headers)")
    return BIN


def test_cpp_shim_schedule(sk):
    out = subprocess.run([_binary(), "--schedule"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count("[PASS]") == 3


@pytest.mark.gpu
def test_cpp_shim_execute(sk):
    out = subprocess.run([_binary(), "--execute"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count("[PASS]") == 3
