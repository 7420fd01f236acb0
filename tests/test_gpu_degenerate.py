"""TriangleMesh::has_degenerate_faces on the device query paths.

reduce_min_over_faces skips degenerate faces only when the mesh's flag is
set (/root/reference/proj/src/kernels.cpp:350,357); otherwise it evaluates
them through the degenerate fallbacks (kernels.cpp:127-134, 151-156,
262-316). The reference's own test builds such a mesh and refreshes the flag
first (test_distance.cpp:278-290); without the refresh it answers ~1.005 at
face 0. intersects_mesh never skips (kernels.cpp:407-432).
"""
import numpy as np
import pytest

import oracle as O
import paper_1808_09571_b200 as T
from conftest import bits

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(O.REF is None, reason="oracle/_ref not built")]


@pytest.fixture(scope="module", autouse=True)
def device():
    T.init(0)
    yield


def _ref_test_mesh():
    return np.array([[0, 0, 1, 1, 0, 1, 2, 0, 1],   # degenerate sliver, closer
                     [0, 0, 0, 1, 0, 0, 0, 1, 0]], float)


def test_reference_case_without_refresh():
    m = _ref_test_mesh()
    p = np.array([[0.2, 0.1, 2.0]])
    for flag, face in ((False, 0), (True, 1)):
        dm = T.Mesh(m).set_has_degenerate_faces(flag)
        d, f = T.points_mesh_distance(p, dm)
        rd, rf = O.ref_queries_mesh_distance_flag(p, m, flag, points=True)
        assert bits(d) == bits(rd) and f[0] == rf[0] == face, (flag, d, f, rd, rf)
    d, f = T.points_mesh_distance(p, T.Mesh(m).set_has_degenerate_faces(False))
    assert f[0] == 0 and abs(d[0] - 1.00498756211) < 1e-9


def _degenerate_soup(rng, n):
    """Random faces, a third of them degenerate in every way the reference
    distinguishes: collinear, repeated vertex, all three equal, and tiny
    (|N|^2 <= 1e-30 while well shaped)."""
    m = rng.uniform(-1, 1, (n, 9))
    k = rng.integers(0, 5, n)
    c = k == 1  # collinear
    t = rng.uniform(-0.5, 1.5, c.sum())[:, None]
    m[c, 6:9] = m[c, 0:3] + t * (m[c, 3:6] - m[c, 0:3])
    r = k == 2  # repeated vertex
    m[r, 3:6] = m[r, 0:3]
    e = k == 3  # one point
    m[e, 3:6] = m[e, 0:3]
    m[e, 6:9] = m[e, 0:3]
    s = k == 4  # tiny but well shaped (edges 1e-9)
    m[s, 3:9] = m[s, 0:3].repeat(2, 0).reshape(-1, 6) + rng.normal(scale=1e-9, size=(s.sum(), 6))
    return m


@pytest.mark.parametrize("n_faces", [500, 20_000])
def test_queries_follow_the_flag(n_faces):
    """Points and segments (incl. zero-length) against a soup with many
    degenerate faces, flag off and on, through the fused (small mesh) and the
    chunked (large mesh) query paths; intersects ignores the flag."""
    rng = np.random.default_rng(n_faces)
    m = _degenerate_soup(rng, n_faces)
    pts = rng.uniform(-1.2, 1.2, (3000, 3))
    segs = np.concatenate([pts, pts + rng.normal(scale=0.3, size=pts.shape)], 1)
    segs[::7, 3:6] = segs[::7, 0:3]
    for flag in (False, True):
        dm = T.Mesh(m).set_has_degenerate_faces(flag)
        for q, is_pt in ((pts, True), (segs, False)):
            d, f = T.points_mesh_distance(q, dm) if is_pt else T.segments_mesh_distance(q, dm)
            rd, rf = O.ref_queries_mesh_distance_flag(q, m, flag, points=is_pt)
            bad = np.flatnonzero((bits(d) != bits(rd)) | (f != rf))
            assert len(bad) == 0, (flag, is_pt, len(bad), q[bad[:3]], d[bad[:3]], rd[bad[:3]], f[bad[:3]], rf[bad[:3]])
        if not flag:  # the degenerate faces really win somewhere (geometry.hpp:75)
            deg = (np.cross(m[:, 3:6] - m[:, 0:3], m[:, 6:9] - m[:, 0:3]) ** 2).sum(1) <= 1e-30
            assert deg[rf[rf != O.U64_MAX].astype(np.int64)].any()
        h, hf = T.segments_mesh_intersects(segs, dm)
        rh, rhf = O.ref_segments_mesh_intersects(segs, m)
        assert np.array_equal(h.astype(bool), rh.astype(bool)) and np.array_equal(hf, rhf)


def test_literal_over_mesh_column_uses_each_records_flag():
    """run_batch(Distance, mesh records, Point / Segment literal): each record
    answers with its own has_degenerate_faces (batch.cpp:44-48)."""
    rng = np.random.default_rng(5)
    objs = [_degenerate_soup(rng, int(k)) for k in rng.integers(1, 60, 40)]
    off = np.cumsum([0] + [len(o) for o in objs]).astype(np.uint64)
    flags = rng.integers(0, 2, len(objs)).astype(bool)
    tab = T.Table(np.concatenate(objs), off).set_has_degenerate_faces(flags)
    for lit, is_pt in ((np.array([0.1, -0.2, 0.3]), True), (np.array([0.1, -0.2, 0.3, -0.4, 0.5, 0.2]), False)):
        d, f = T.literal_table_eval(T.OP_DISTANCE, lit, tab)
        for o, mo in enumerate(objs):
            rd, rf = O.ref_queries_mesh_distance_flag(lit[None, :], mo, flags[o], points=is_pt)
            assert bits(d[o]) == bits(rd[0]) and f[o] == rf[0], (o, flags[o], d[o], rd, f[o], rf)


@pytest.mark.parametrize("mesh", ["soup", "sphere"])
def test_fused_query_paths_follow_the_flag(mesh):
    """40,000 queries against one small mesh: the fused kernel (the whole mesh
    in one chunk, q_fused_kernel), flag cleared and set, on a soup with
    degenerate faces and on a clean sphere; bit-exact against the reference."""
    rng = np.random.default_rng(77)
    m = _degenerate_soup(rng, 500) if mesh == "soup" else T.unit_sphere(1000)
    pts = rng.uniform(-1.2, 1.2, (40_000, 3))
    segs = np.concatenate([pts, pts + rng.normal(scale=0.3, size=pts.shape)], 1)
    segs[::7, 3:6] = segs[::7, 0:3]
    for flag in (False, True):
        dm = T.Mesh(m).set_has_degenerate_faces(flag)
        for q, is_pt in ((pts, True), (segs, False)):
            d, f = T.points_mesh_distance(q, dm) if is_pt else T.segments_mesh_distance(q, dm)
            rd, rf = O.ref_queries_mesh_distance_flag(q, m, flag, points=is_pt)
            bad = np.flatnonzero((bits(d) != bits(rd)) | (f != rf))
            assert len(bad) == 0, (mesh, flag, is_pt, len(bad), q[bad[:3]], d[bad[:3]], rd[bad[:3]], f[bad[:3]],
                                   rf[bad[:3]])
