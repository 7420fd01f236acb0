"""bench.py output contract, checked on CPU through the reference arm
(--impl reference runs only the CPU reference; the GPU arm prints the same
keys plus roofline / clocks / gpu_launches, exercised on the B200)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
from conftest import ROOT


@pytest.mark.skipif(O.C is None, reason="oracle not built")
def test_reference_arm_prints_one_contract_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "2", "--warmup", "1", "--ref-rows", "4"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "pairs/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1 and d["dtype"] == "f64"
    assert d["vs_baseline"] is None and d["scaling"] == "weak"
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["cores"] >= 1 and cb["kind"] in ("reference", "port") and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert "workload" in d["config"]


def test_reference_arm_non_zero_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--config", "c1",
                        "--steps", "1", "--warmup", "0", "--ref-rows", "1"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""


@pytest.mark.skipif(O.REF is None, reason="oracle/_ref not built")
def test_reference_arm_never_loads_the_product():
    """The reference arm builds its inputs with the reference's generators
    (oracle/_ref) and must not import paper_1808_09571_b200 or map its .so."""
    code = ("import sys, runpy; sys.argv = ['bench.py', '--impl', 'reference', '--config', 'c1', '--steps', '1', "
            "'--warmup', '0', '--ref-rows', '2']; runpy.run_path('bench.py', run_name='__main__'); "
            "maps = open('/proc/self/maps').read(); "
            "assert 'paper_1808_09571_b200' not in sys.modules, 'product imported'; "
            "assert 'libtindb_b200' not in maps, 'product library mapped'")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]


@pytest.mark.skipif(O.REF is None, reason="oracle/_ref not built")
def test_both_arms_print_the_same_config():
    import argparse

    import bench
    for cfg in ("c1", "c2"):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", cfg,
                            "--steps", "1", "--warmup", "0", "--ref-rows", "1"],
                           capture_output=True, text=True, timeout=600, cwd=ROOT)
        assert r.returncode == 0, r.stderr
        ref_cfg = json.loads(r.stdout.strip().splitlines()[-1])["config"]
        wl = bench.workload(cfg, None, 100_000)
        wl.build(bench.ProductGen())
        args = argparse.Namespace(mode="full", scaling="weak")
        assert ref_cfg == bench.config_of(args, wl, 1)


@pytest.mark.skipif(O.REF is None, reason="oracle/_ref not built")
def test_generators_of_both_arms_are_bit_identical():
    import bench
    P, R = bench.ProductGen(), bench.ReferenceGen()
    for f, a in (("terrain", (64, 32, 20.0, 42)), ("unit_sphere", (10000,)), ("ore_body", (1000,))):
        x, y = getattr(P, f)(*a), getattr(R, f)(*a)
        assert np.array_equal(x.view(np.uint64), y.view(np.uint64)), f
    assert np.array_equal(P.drills(100, 42).view(np.uint64), R.drills(100, 42).view(np.uint64))


@pytest.mark.timeout(300)
def test_bench_gpus_2_spawns_two_ranks_that_cover_the_job():
    """`bench.py --gpus 2` with no launcher starts two ranks itself
    (torch.distributed.run on 127.0.0.1); under gloo the plan-only mode checks
    that the ranks' unit ranges tile each step, weak and strong."""
    for scaling in ("weak", "strong"):
        env = dict(os.environ, TDB_BENCH_BACKEND="gloo")
        env.pop("WORLD_SIZE", None)
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--plan-only",
                            "--config", "c1", "--batch-rows", "2048", "--steps", "3", "--warmup", "1",
                            "--scaling", scaling], capture_output=True, text=True, timeout=280, cwd=ROOT, env=env)
        assert r.returncode == 0, r.stderr[-3000:]
        d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
        assert d["n_gpus"] == 2 and d["scaling"] == scaling
        n, bu = d["n_units"], d["batch_units"]
        r0, r1 = d["spans"]
        for s in range(3):
            (a0, a1), (b0, b1) = r0[s], r1[s]
            if scaling == "strong":  # both ranks split batch s = warmup + s
                b = (1 + s) % (n // bu)
                assert (a0, a1, b1) == (b * bu, b0, (b + 1) * bu) and a0 < a1 < b1
            else:  # rank r takes whole batch (warmup + s) * 2 + r
                assert (a0, a1) == ((((1 + s) * 2) % (n // bu)) * bu, (((1 + s) * 2) % (n // bu)) * bu + bu)
                assert (b0, b1) == ((((1 + s) * 2 + 1) % (n // bu)) * bu, (((1 + s) * 2 + 1) % (n // bu)) * bu + bu)
        assert d["combined"] == [float(r0[0][0]) if r0[0][0] <= r1[0][0] else float(r1[0][0]),
                                 0 if r0[0][0] <= r1[0][0] else 1]


def test_bench_rejects_world_size_mismatch():
    env = dict(os.environ, RANK="0", WORLD_SIZE="2", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--impl", "reference",
                        "--config", "c1", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr
