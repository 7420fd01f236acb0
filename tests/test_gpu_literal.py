"""GPU parity: run_batch with a Segment / Point literal over a mesh column
(batch.cpp:44-48, :59) and Volume over a mesh column, against the
reference's own distance_to_mesh / intersects_mesh (oracle/_ref)."""
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


def _table(rng, n=40):
    meshes = []
    for k in range(n):
        ft = [10, 100, 1000][k % 3]
        m = T.unit_sphere(ft) * rng.uniform(2, 10) + rng.uniform(0, 100, 3).tolist() * 3
        if k % 7 == 3:
            m = np.concatenate([m[:5], np.tile([[1, 1, 1, 2, 2, 2, 3, 3, 3]], (3, 1)), m[5:]])  # degenerate faces
        meshes.append(m)
    meshes.append(np.zeros((0, 9)))  # an empty record
    off = np.concatenate([[0], np.cumsum([len(m) for m in meshes])])
    return meshes, T.Table(np.concatenate(meshes), off)


@pytest.mark.skipif(O.REF is None, reason="reference not built")
def test_segment_and_point_literal_against_mesh_column():
    rng = np.random.default_rng(5)
    meshes, tab = _table(rng)
    segs = [np.array([10.0, 10, 10, 90, 90, 90]), np.array([50.0, 50, -5, 50, 50, 120]),
            np.array([30.0, 30, 30, 30, 30, 30])]  # the last is zero-length: a point query
    for s in segs:
        d, f = T.literal_table_eval(T.OP_DISTANCE, s, tab)
        h, hf = T.literal_table_eval(T.OP_INTERSECTS, s, tab)
        for i, m in enumerate(meshes):
            rd, rf = O.ref_segments_mesh_distance(s.reshape(1, 6), m)
            assert bits(d[i]) == bits(rd[0]) and f[i] == rf[0], (i, d[i], rd[0])
            rh, rhf = O.ref_segments_mesh_intersects(s.reshape(1, 6), m)
            assert h[i] == bool(rh[0]) and hf[i] == rhf[0], i
    p = np.array([40.0, 60.0, 20.0])
    d, f = T.literal_table_eval(T.OP_DISTANCE, p, tab)
    for i, m in enumerate(meshes):
        rd, rf = O.ref_points_mesh_distance(p.reshape(1, 3), m)
        assert bits(d[i]) == bits(rd[0]) and f[i] == rf[0], i
