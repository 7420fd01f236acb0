"""The C++ drop-in shim (include/tindb_b200/kernels.hpp) on the reference's
own types and run_batch dispatch: tests/cpp/shim_test.cpp, built by
`make shimtest` against the reference headers and linked with the reference
sources (oracle/_ref) and libtindb_b200.so."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
BIN = os.path.join(ROOT, "build", "shim_test")


@pytest.mark.skipif(not os.path.exists(BIN), reason="build/shim_test not built (needs /root/reference)")
def test_cpp_shim_against_reference_dispatch():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "SHIM OK" in r.stdout
