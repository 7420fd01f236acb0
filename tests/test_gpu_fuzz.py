"""GPU fuzz parity: seeded adversarial meshes against the CPU oracle
(oracle/tindb_oracle.c, pinned bit-for-bit to the reference build).

Each case builds two small meshes whose closest / crossing pairs sit where
the filter's error bound matters: near-parallel and coplanar faces, shared
vertices and edges, slivers near the 1e-30 degeneracy threshold, exact
duplicates (ties), and scales from 1e-3 to 1e4 at offsets up to 1e6. Every
answer must be bit-identical: distance bits, lowest pair, hit, lowest hit.
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


def _rot(rng):
    q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    return q


def _place(m, R, t, s):
    v = m.reshape(-1, 3) @ R.T * s + t
    return v.reshape(-1, 9)


def _case(rng):
    """(a, b) for one adversarial configuration."""
    kind = rng.integers(0, 6)
    n = int(rng.integers(20, 260))
    base = rng.uniform(-1, 1, (n, 9))
    if kind == 0:  # two nearly parallel sheets, gap g
        g = 10.0 ** rng.uniform(-9, -1)
        a = base.copy()
        a[:, 2::3] = rng.uniform(-1e-3, 1e-3, (n, 3))
        b = a.copy() + rng.normal(scale=0.05, size=a.shape)
        b[:, 2::3] = g + rng.uniform(-1e-9, 1e-9, (n, 3))
    elif kind == 1:  # coplanar overlapping soups
        a = base.copy()
        a[:, 2::3] = 0.0
        b = rng.uniform(-1, 1, (n, 9))
        b[:, 2::3] = 0.0
    elif kind == 2:  # shared vertices / edges: b reuses a's vertices
        a = base
        b = a[rng.permutation(n)].copy()
        b[:, 6:9] = rng.uniform(-1, 1, (n, 3))
    elif kind == 3:  # slivers near the degeneracy threshold
        a = base
        b = rng.uniform(-1, 1, (n, 9))
        eps = 10.0 ** rng.uniform(-16, -14, n)
        b[:, 6:9] = b[:, 0:3] + (b[:, 3:6] - b[:, 0:3]) * 0.5 + eps[:, None] * rng.normal(size=(n, 3))
    elif kind == 4:  # exact duplicates: every minimum tied
        a = base
        b = np.concatenate([a[: n // 2], a[: n // 2]]) + np.array([0.0, 0.0, 2.0] * 3)
    else:  # near-touching clusters
        a = base
        b = rng.uniform(-0.3, 0.3, (n, 9)) + np.tile(a.reshape(n, 3, 3).mean(1), 3) + rng.normal(
            scale=1e-3, size=(n, 9))
    R = _rot(rng)
    s = 10.0 ** rng.uniform(-3, 4)
    t = rng.uniform(-1, 1, 3) * 10.0 ** rng.uniform(0, 6)
    return _place(a, R, t, s), _place(b, R, t, s)


@pytest.mark.parametrize("seed", range(24))
def test_adversarial_meshes_bit_exact(seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(25):
        a, b = _case(rng)
        r = T.mesh_mesh_distance(a, b)
        d, p, found, wa, wb = O.mesh_mesh_distance(a, b)
        assert bits(r.distance) == bits(d), (seed, r.distance, d)
        assert (r.pair_index if r.pair_index is not None else O.U64_MAX) == p
        h = T.mesh_mesh_intersects(a, b)
        hit, hp = O.mesh_mesh_intersects(a, b)
        assert h.hit == hit and (h.pair_index if h.hit else O.U64_MAX) == hp


def test_adversarial_table_and_cull_mode():
    rng = np.random.default_rng(77)
    recs, q = [], None
    for k in range(30):
        a, b = _case(rng)
        if q is None:
            q = b
        recs.append(a)
    # records in q's frame: shift them near q
    off = np.concatenate([[0], np.cumsum([len(r) for r in recs])])
    tab = T.Table(np.concatenate(recs), off)
    d, p = T.table_eval(T.OP_DISTANCE, tab, T.Mesh(q))
    h, hp = T.table_eval(T.OP_INTERSECTS, tab, T.Mesh(q))
    T.set_mode(T.MODE_CULL)
    try:
        dc, pc = T.table_eval(T.OP_DISTANCE, tab, T.Mesh(q))
    finally:
        T.set_mode(T.MODE_FULL)
    assert np.array_equal(bits(d), bits(dc)) and np.array_equal(p, pc)
    for i, r in enumerate(recs):
        rd, rp, *_ = O.mesh_mesh_distance(r, q)
        assert bits(d[i]) == bits(rd) and p[i] == rp, i
        rh, rhp = O.mesh_mesh_intersects(r, q)
        assert h[i] == rh and hp[i] == rhp, i


@pytest.mark.parametrize("seed", range(6))
def test_adversarial_segments_and_points_bit_exact(seed):
    """distance_to_mesh / intersects_mesh with segments lying in, grazing or
    piercing the faces' planes, and zero-length segments."""
    rng = np.random.default_rng(2000 + seed)
    for _ in range(10):
        a, b = _case(rng)
        m = a
        tri = m[rng.integers(0, len(m), 400)].reshape(-1, 3, 3)
        w = rng.dirichlet([1, 1, 1], len(tri))
        p_in = np.einsum("ni,nij->nj", w, tri)  # points on faces
        nrm = np.cross(tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0])
        nrm /= np.linalg.norm(nrm, axis=1, keepdims=True) + 1e-300
        edge = tri[:, 1] - tri[:, 0]
        k = rng.integers(0, 4, len(tri))
        lift = (10.0 ** rng.uniform(-12, -2, len(tri)))[:, None] * np.abs(m).max()
        d = np.where((k == 0)[:, None], edge, nrm)  # in-plane or normal
        p0 = p_in + np.where((k == 1)[:, None], -lift * nrm, lift * nrm * (k == 2)[:, None])
        p1 = p0 + d * rng.uniform(0.1, 2.0, (len(tri), 1))
        p1[k == 3] = p0[k == 3]  # zero-length: a point query
        segs = np.concatenate([p0, p1], axis=1)
        dd, ff = T.segments_mesh_distance(segs, m)
        rd, rf = O.segments_mesh_distance(segs, m)
        assert np.array_equal(bits(dd), bits(rd)) and np.array_equal(ff, rf), seed
        hh, hf = T.segments_mesh_intersects(segs, m)
        rh, rhf = O.segments_mesh_intersects(segs, m)
        assert np.array_equal(hh.astype(bool), rh.astype(bool)) and np.array_equal(hf, rhf), seed
        pd, pf = T.points_mesh_distance(p0, m)
        rpd, rpf = O.points_mesh_distance(p0, m)
        assert np.array_equal(bits(pd), bits(rpd)) and np.array_equal(pf, rpf), seed
