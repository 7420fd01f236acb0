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


ENGINE = os.path.join(ROOT, "build", "engine_test")


@pytest.mark.skipif(not os.path.exists(ENGINE), reason="build/engine_test not built (needs /root/reference)")
def test_sql_route_through_reference_engine():
    """SQL statements through the reference engine with
    run_batch routed to the device give the reference's rendered text cell
    for cell, and the snapshot's device columns are built once."""
    r = subprocess.run([ENGINE], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ENGINE OK" in r.stdout


REFUNIT = os.path.join(ROOT, "build", "ref_unit_tests")


@pytest.mark.skipif(not os.path.exists(REFUNIT), reason="build/ref_unit_tests not built (needs /root/reference)")
def test_reference_unit_tests_on_the_device_engine():
    """The reference's own unit tests for the replaced entry points
    (tests/test_batch.cpp, test_volume.cpp, test_distance.cpp,
    test_intersect.cpp, test_geometry.cpp, test_store.cpp, test_sqlfe.cpp,
    unmodified) with run_batch (also inside the reference engine, for
    test_sqlfe), mesh_volume, distance_to_mesh, intersects_mesh, parse_wkt
    and the table loaders routed to the device shim: every case passes (the
    primitive-level cases in those files run the reference's own
    primitives)."""
    r = subprocess.run([REFUNIT], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "113 test cases, 0 failed" in r.stdout, r.stdout
