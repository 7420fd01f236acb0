"""Full-size parity: the GPU answer on the BASELINE
configurations against the AABB-pruned exact CPU oracle.

The pruned oracle evaluates the reference composition on every pair whose
exact distance can be <= ub, so with ub = the GPU's reported distance it
returns the true lexicographic minimum (distance, pair) of the whole job:
equal to the GPU's iff the GPU's answer is the reference's (a GPU answer
that were too large would be undercut, one that were not a real pair could
not be reproduced).
"""
import numpy as np
import pytest

import oracle as O
import paper_1808_09571_b200 as T
from conftest import bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def device():
    T.init(0)
    yield


@pytest.fixture(scope="module")
def c2():
    return T.Mesh(T.terrain(1024, 512, 20.0, 42)), T.terrain(1024, 512, 20.0, 42), T.ore_body(1_000_000)


def test_c2_full_job_distance_bitexact(c2):
    """1,048,576 x 1,310,720 = 1.37e12 pairs, every one evaluated."""
    dA, ter, ore = c2
    r = T.mesh_mesh_distance(dA, T.Mesh(ore))
    st = T.last_stats()
    assert st["pairs"] == len(ter) * len(ore)
    d, p, found, wa, wb = O.mesh_mesh_distance_pruned(ter, ore, r.distance)
    assert found and bits(r.distance) == bits(d) and r.pair_index == p
    assert np.array_equal(bits(np.array(r.closest_on_a)), bits(wa))
    assert np.array_equal(bits(np.array(r.closest_on_b)), bits(wb))


def test_c3_full_job_intersects_no_hit():
    """1,310,720 x 1,310,720 concentric (0.9x): overlapping AABBs, no hit."""
    s = T.unit_sphere(1_000_000)
    h = T.mesh_mesh_intersects(s, s * 0.9)
    assert T.last_stats()["pairs"] == len(s) ** 2
    assert not h.hit
    assert O.mesh_mesh_intersects_pruned(s, s * 0.9) == (False, O.U64_MAX)


def test_c3_variant_with_hits_lowest_pair():
    s = T.unit_sphere(100_000)
    b = T.translate(s * 0.999, 0.3, 0.05, 0.0)
    h = T.mesh_mesh_intersects(s, b)
    hit, hp = O.mesh_mesh_intersects_pruned(s, b)
    assert h.hit == hit and h.pair_index == hp
    r = T.mesh_mesh_distance(s, b)
    d, p, found, *_ = O.mesh_mesh_distance_pruned(s, b, r.distance)
    assert found and bits(r.distance) == bits(d) and r.pair_index == p


def test_c5_answer_shard():
    """C5 (8,388,608^2): the shard of rows holding the global answer."""
    s = T.unit_sphere(10_000_000)
    b = T.translate(s, 2.5, 0.0, 0.0)
    d, p, found, *_ = O.mesh_mesh_distance_pruned(s, b, 0.5)
    assert found and d == 0.5
    i = p // len(b)
    r0 = (i // 65536) * 65536
    r = T.mesh_mesh_distance(T.Mesh(s), T.Mesh(b), rows=(r0, min(len(s), r0 + 65536)))
    assert bits(r.distance) == bits(d) and r.pair_index == p


def test_c4_table_records_bitexact():
    """C4 shape (1,280-face records vs the 81,920-face query), 96 records."""
    q = T.ore_body(100_000)
    base = T.unit_sphere(1000)
    rng = np.random.default_rng(42)
    n = 96
    scale = rng.uniform(2.0, 10.0, n)
    ctr = np.stack([rng.uniform(300, 700, n), rng.uniform(300, 700, n), rng.uniform(-350, -50, n)], 1)
    objs = [T.translate(base * scale[k], *ctr[k]) for k in range(n)]
    off = np.arange(n + 1, dtype=np.uint64) * len(base)
    tab = T.Table(np.concatenate(objs), off)
    d, pr = T.table_eval(T.OP_DISTANCE, tab, T.Mesh(q))
    h, hp = T.table_eval(T.OP_INTERSECTS, tab, T.Mesh(q))
    assert h.any() and not h.all()
    for k in range(n):
        od, op_, found, *_ = O.mesh_mesh_distance_pruned(objs[k], q, d[k])
        assert found and bits(od) == bits(d[k]) and op_ == pr[k], k
        ohit, ohp = O.mesh_mesh_intersects_pruned(objs[k], q)
        assert ohit == h[k] and ohp == hp[k], k
