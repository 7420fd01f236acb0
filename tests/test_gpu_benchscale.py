"""Parity at the sizes bench.py reports (VERDICT r1 "bench-scale parity").

* C4: the bench's own 100,000-record table (bench.py TableWorkload: 100,000
  unit_sphere(1000) records x U[2,10] + U(box) against the 81,920-face ore
  body), both ops. The whole table is evaluated on the device (CULL mode,
  whose answers are FULL mode's), then 2,000 random records, every hit
  record and the global-minimum record again in FULL mode (the bench's mode),
  each against the AABB-pruned exact oracle.
* C3 stress: 1,310,720-face sphere vs its 0.999x copy rotated 0.37 rad about
  (1, 2, 3) (surfaces 1e-3 apart, no hit) — the full job.
* C5 shape: two 2,097,152-face spheres offset 2.5 (answer exactly 0.5),
  the full 4.4e12-pair job.
"""
import numpy as np
import pytest

import bench
import oracle as O
import paper_1808_09571_b200 as T
from conftest import bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def device():
    T.init(0)
    yield
    T.set_mode(T.MODE_FULL)


def test_c4_bench_table_parity():
    wl = bench.workload("c4", None, 100_000)
    wl.build(bench.ProductGen())
    nf, n = wl.nf, wl.n_objects
    off = np.arange(n + 1, dtype=np.uint64) * nf
    tab, q = T.Table(wl.tab, off), T.Mesh(wl.Q)
    T.set_mode(T.MODE_CULL)
    try:
        d_all, p_all = T.table_eval(T.OP_DISTANCE, tab, q)
        h_all, hp_all = T.table_eval(T.OP_INTERSECTS, tab, q)
    finally:
        T.set_mode(T.MODE_FULL)
    assert h_all.any() and not h_all.all()
    rng = np.random.default_rng(7)
    sample = set(rng.choice(n, 2000, replace=False).tolist())
    sample |= set(np.flatnonzero(h_all).tolist())
    sample.add(int(np.argmin(d_all)))
    checked = 0
    for o in sorted(sample):
        d, p = T.table_eval(T.OP_DISTANCE, tab, q, objects=(o, o + 1))
        h, hp = T.table_eval(T.OP_INTERSECTS, tab, q, objects=(o, o + 1))
        assert bits(d[0]) == bits(d_all[o]) and p[0] == p_all[o], o  # FULL == CULL
        assert h[0] == h_all[o] and hp[0] == hp_all[o], o
        rec = wl.tab[o * nf:(o + 1) * nf]
        od, op_, found, *_ = O.mesh_mesh_distance_pruned(rec, wl.Q, d[0])
        assert found and bits(od) == bits(d[0]) and op_ == p[0], (o, od, d[0], op_, p[0])
        ohit, ohp = O.mesh_mesh_intersects_pruned(rec, wl.Q)
        assert ohit == h[0] and ohp == hp[0], (o, ohit, ohp, h[0], hp[0])
        checked += 1
    print(f"C4 bench table: {h_all.sum()} hit records, min {d_all.min()} at record {int(np.argmin(d_all))}, "
          f"{checked} records checked against the pruned oracle")


def test_c3_stress_full_job_no_hit():
    wl = bench.workload("c3s", None, 0)
    wl.build(bench.ProductGen())
    h = T.mesh_mesh_intersects(wl.A, wl.B)
    assert T.last_stats()["pairs"] == len(wl.A) * len(wl.B)
    assert not h.hit
    assert O.mesh_mesh_intersects_pruned(wl.A, wl.B) == (False, O.U64_MAX)
    r = T.mesh_mesh_distance(wl.A[:65536], wl.B)  # a distance shard of the same pair: surfaces 1e-3 apart
    d, p, found, *_ = O.mesh_mesh_distance_pruned(wl.A[:65536], wl.B, r.distance)
    assert found and bits(r.distance) == bits(d) and r.pair_index == p


@pytest.mark.slow
def test_c5_shape_full_job():
    s = T.unit_sphere(2_000_000)          # octahedron L9: 2,097,152 faces
    assert len(s) == 2_097_152
    b = bench.translate(s, 2.5, 0.0, 0.0)
    r = T.mesh_mesh_distance(T.Mesh(s), T.Mesh(b))
    assert T.last_stats()["pairs"] == len(s) * len(b)
    d, p, found, *_ = O.mesh_mesh_distance_pruned(s, b, r.distance)
    assert found and d == 0.5 and bits(r.distance) == bits(d) and r.pair_index == p
