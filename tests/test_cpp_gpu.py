"""Runs the C++ drop-in check (tests/cpp/test_contract.cpp): reference-style
gridjit C++ code compiled against include/tt/gridjit_b200.hpp, executed on
the GPU (manual driver flow, cuda_launch facade, trace_t05 bit-exact)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_contract_program(gpu):
    exe = os.path.join(ROOT, "tests", "cpp", "test_contract")
    if not os.path.exists(exe):
        import __graft_entry__
        __graft_entry__.build_cpp_tests()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
