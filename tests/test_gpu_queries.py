"""Segment x mesh and point x mesh on the device (the paper's drill-hole
workload) against the reference's own distance_to_mesh / intersects_mesh
(golden vectors from oracle/_ref, tests/golden/make_golden.py) and the C
oracle: distances bit-for-bit, lowest face indices and hits exactly."""
import numpy as np
import pytest

import oracle as O
import paper_1808_09571_b200 as T
from conftest import GOLDEN, bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def device():
    T.init(0)
    yield


@pytest.fixture(scope="module")
def golden():
    import os
    return dict(np.load(os.path.join(GOLDEN, "queries.npz")))


@pytest.mark.parametrize("ore", ["ore512", "ore20480"])
def test_segments_distance_bitwise(golden, ore):
    d, f = T.segments_mesh_distance(golden["segments"], golden[f"{ore}/mesh"])
    assert np.array_equal(bits(d), bits(golden[f"{ore}/seg_dist"]))
    assert np.array_equal(f, golden[f"{ore}/seg_face"])


@pytest.mark.parametrize("ore", ["ore512", "ore20480"])
def test_points_distance_bitwise(golden, ore):
    d, f = T.points_mesh_distance(golden["points"], golden[f"{ore}/mesh"])
    assert np.array_equal(bits(d), bits(golden[f"{ore}/pt_dist"]))
    assert np.array_equal(f, golden[f"{ore}/pt_face"])


@pytest.mark.parametrize("ore", ["ore512", "ore20480"])
def test_segments_intersects_exact(golden, ore):
    h, f = T.segments_mesh_intersects(golden["segments"], golden[f"{ore}/mesh"])
    assert np.array_equal(h, golden[f"{ore}/seg_hit"])
    assert np.array_equal(f, golden[f"{ore}/seg_hit_face"])


def test_paper_scale_drills_vs_oracle():
    """100k drills (make_drills, seed 42) x the 1,280-face ore: every answer
    against the C oracle (pinned to the reference)."""
    drills = T.drills(100_000, 42)
    ore = T.ore_body(1000)
    d, f = T.segments_mesh_distance(drills, ore)
    od, of = O.segments_mesh_distance(drills, ore)
    assert np.array_equal(bits(d), bits(od)) and np.array_equal(f, of)
    h, hf = T.segments_mesh_intersects(drills, ore)
    oh, ohf = O.segments_mesh_intersects(drills, ore)
    assert np.array_equal(h, oh) and np.array_equal(hf, ohf)
    assert 0 < h.sum() < len(h)


def test_fused_and_chunked_paths_agree_resident():
    """>= 2 x SMs tiles with a one-chunk mesh take the fused kernel; a larger
    mesh takes the chunked filter/verify path; both match the oracle."""
    drills = T.drills(60_000, 7)
    q = T.Queries(drills)
    small, big = T.ore_body(1000), T.ore_body(20_000)  # 1,280 (fused) / 20,480 faces (chunked)
    for ore in (small, big):
        d, f = T.queries_mesh_distance(q, ore)
        st = T.last_stats()
        od, of = O.segments_mesh_distance(drills, ore)
        assert np.array_equal(bits(d), bits(od)) and np.array_equal(f, of)
        assert st["pairs"] == len(drills) * len(ore)
        h, hf = T.queries_mesh_intersects(q, ore)
        oh, ohf = O.segments_mesh_intersects(drills, ore)
        assert np.array_equal(h, oh) and np.array_equal(hf, ohf)
    pts = T.Queries(drills[:, :3].copy(), T.QUERY_POINTS)
    d, f = T.queries_mesh_distance(pts, small)
    od, of = O.points_mesh_distance(drills[:, :3].copy(), small)
    assert np.array_equal(bits(d), bits(od)) and np.array_equal(f, of)
    with pytest.raises(ValueError):
        T.queries_mesh_intersects(pts, small)  # intersects takes segments


def test_queries_with_degenerate_faces_and_ties():
    s = T.unit_sphere(80)
    mesh = np.concatenate([s[:10], np.tile([[0, 0, 0, 1, 1, 1, 2, 2, 2]], (3, 1)), s[:10], s[10:]])  # dups + slivers
    rng = np.random.default_rng(3)
    segs = rng.uniform(-2, 2, (500, 6))
    segs[::17, 3:] = segs[::17, :3]
    pts = rng.uniform(-2, 2, (500, 3))
    d, f = T.segments_mesh_distance(segs, mesh)
    od, of = O.segments_mesh_distance(segs, mesh)
    assert np.array_equal(bits(d), bits(od)) and np.array_equal(f, of)
    pd, pf = T.points_mesh_distance(pts, mesh)
    opd, opf = O.points_mesh_distance(pts, mesh)
    assert np.array_equal(bits(pd), bits(opd)) and np.array_equal(pf, opf)
    h, hf = T.segments_mesh_intersects(segs, mesh)
    oh, ohf = O.segments_mesh_intersects(segs, mesh)
    assert np.array_equal(h, oh) and np.array_equal(hf, ohf)


def test_empty_inputs():
    s = T.unit_sphere(80)
    d, f = T.segments_mesh_distance(np.zeros((0, 6)), s)
    assert len(d) == 0
    d, f = T.points_mesh_distance(np.ones((3, 3)), np.zeros((0, 9)))
    assert np.isinf(d).all() and (f == O.U64_MAX).all()
