"""Parity of the shared-candidate distance filter.

FULL mode evaluates each distinct vertex / edge of a 64-face B block and each
distinct vertex / edge of a 128-face A tile once (filter_kernel<false>,
vertex_kernel, edge_kernel); CULL mode keeps per-face A candidates
(filter_kernel<true>). These cases stress what the sharing depends on:
vertices shared bitwise between faces, shared edges seen in opposite
directions, degenerate faces inside blocks and tiles (excluded from the
lists), store sizes that are not multiples of 64 / 128, pure soups (nothing
shared), row selections that cut a tile, and tables whose records straddle
tiles. Every answer must be bit-identical to the CPU oracle.
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
    T.set_mode(T.MODE_FULL)


def _rot(rng):
    q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    return q


def _mixed(rng, n_sphere=1000, n_soup=300):
    """A subdivided sphere (shared vertices / edges), a third of its faces
    with reversed orientation (shared edges in both directions), degenerate
    faces sprinkled in, and a random soup (nothing shared), shuffled in runs."""
    s = T.unit_sphere(n_sphere)
    s = s[: int(rng.integers(len(s) * 2 // 3, len(s)))].copy()
    flip = rng.random(len(s)) < 0.33
    s[flip] = s[flip][:, [0, 1, 2, 6, 7, 8, 3, 4, 5]]
    soup = rng.uniform(-1, 1, (n_soup, 9)) * 0.2 + 0.9
    deg = s[rng.integers(0, len(s), 25)].copy()
    deg[:, 6:9] = deg[:, 0:3]  # collapsed: exactly degenerate
    parts = [s, soup, deg]
    m = np.concatenate(parts)
    # shuffle in runs of 5..40 faces so blocks mix shared and unshared faces
    cuts = np.sort(rng.choice(np.arange(1, len(m)), size=len(m) // 20, replace=False))
    runs = np.split(m, cuts)
    rng.shuffle(runs)
    m = np.concatenate(runs)
    v = m.reshape(-1, 3) @ _rot(rng).T
    return np.ascontiguousarray(v.reshape(-1, 9))


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("mode", ["full", "cull"])
def test_mixed_meshes_bit_exact(seed, mode):
    rng = np.random.default_rng(seed)
    a = _mixed(rng)
    b = np.ascontiguousarray(_mixed(rng) * rng.uniform(0.3, 1.5) + np.tile(rng.uniform(1.5, 3.0, 3), 3))
    T.set_mode(T.MODE_FULL if mode == "full" else T.MODE_CULL)
    try:
        r = T.mesh_mesh_distance(T.Mesh(a), T.Mesh(b))
    finally:
        T.set_mode(T.MODE_FULL)
    assert T.last_stats()["pairs"] == len(a) * len(b) > 98304  # the filter path, not the direct kernel
    d, p, found, *_ = O.mesh_mesh_distance(a, b)
    assert found and bits(r.distance) == bits(d) and r.pair_index == p, (r, d, p)


@pytest.mark.parametrize("seed", [4, 5])
def test_touching_and_intersecting_mixed(seed):
    """b overlaps a (distance 0 through piercing pairs) and, separately,
    touches it at a shared vertex: the lowest pair among the exact zeros."""
    rng = np.random.default_rng(seed)
    a = _mixed(rng)
    shift = np.array([0.35, 0.0, 0.0] * 3)
    b = np.ascontiguousarray(a[rng.permutation(len(a))][:900] * 0.8 + shift)
    r = T.mesh_mesh_distance(T.Mesh(a), T.Mesh(b))
    d, p, found, *_ = O.mesh_mesh_distance(a, b)
    assert found and bits(r.distance) == bits(d) and r.pair_index == p
    k = next(i for i in range(len(a)) if not np.array_equal(a[i, 6:9], a[i, 0:3]))  # not a collapsed face
    c = np.ascontiguousarray(np.concatenate([b + 5.0, a[k:k + 1]]))  # a non-degenerate face of a, repeated
    r = T.mesh_mesh_distance(T.Mesh(a), T.Mesh(c))
    d, p, found, *_ = O.mesh_mesh_distance(a, c)
    assert found and d == 0.0 and bits(r.distance) == bits(d) and r.pair_index == p


def test_pure_soups_and_odd_sizes():
    rng = np.random.default_rng(11)
    for na, nb in [(129, 1000), (1000, 65), (257, 257), (641, 383)]:
        a = rng.uniform(-1, 1, (na, 9))
        b = rng.uniform(-1, 1, (nb, 9)) + 2.2
        r = T.mesh_mesh_distance(T.Mesh(a), T.Mesh(b))
        d, p, found, *_ = O.mesh_mesh_distance(a, b)
        assert found and bits(r.distance) == bits(d) and r.pair_index == p, (na, nb)


def test_row_selections_cutting_tiles():
    """rows that start / end inside 128-face tiles: a tile's distinct edges
    and vertices may come from rows outside the selection (a lower filter
    minimum only widens the band), the answer must not change."""
    rng = np.random.default_rng(21)
    a = _mixed(rng, 4000, 500)
    b = np.ascontiguousarray(_mixed(rng) + 2.4)
    ma, mb = T.Mesh(a), T.Mesh(b)
    for r0, r1 in [(37, 1500), (128, 129), (1, 4096), (1000, len(a) - 3)]:
        r = T.mesh_mesh_distance(ma, mb, rows=(r0, r1))
        d, p, found, *_ = O.mesh_mesh_distance(a, b, rows=(r0, r1, 1))
        assert found and bits(r.distance) == bits(d) and r.pair_index == p, (r0, r1, r, d, p)


def test_table_records_straddling_tiles():
    rng = np.random.default_rng(31)
    recs = [_mixed(rng, 100, int(rng.integers(1, 90)))[: int(rng.integers(1, 300))] + np.tile(rng.uniform(-3, 3, 3), 3)
            for _ in range(40)]
    tab = np.ascontiguousarray(np.concatenate(recs))
    off = np.concatenate([[0], np.cumsum([len(x) for x in recs])]).astype(np.uint64)
    q = np.ascontiguousarray(_mixed(rng) * 0.5)
    d_all, p_all = T.table_eval(T.OP_DISTANCE, T.Table(tab, off), T.Mesh(q))
    for o, rec in enumerate(recs):
        d, p, found, *_ = O.mesh_mesh_distance(np.ascontiguousarray(rec), q)
        if not found:
            assert p_all[o] == O.U64_MAX
            continue
        assert bits(d_all[o]) == bits(d) and p_all[o] == p, (o, d_all[o], d, p_all[o], p)


def test_feature_counts():
    s = T.Mesh(T.unit_sphere(100_000))  # 81,920 faces, subdivision order
    c = s.feature_counts()
    assert c["faces"] == 81920
    assert 0.5 < c["vertices"] / c["faces"] < 1.0 and 1.5 < c["edges"] / c["faces"] < 2.0
    assert c["tile_edges"] < 2.2 * 81920 and c["tile_vertices"] < 1.2 * 81920
    soup = T.Mesh(np.random.default_rng(0).uniform(-1, 1, (1000, 9)))
    c = soup.feature_counts()
    assert c == {"faces": 1000, "vertices": 3000, "edges": 3000, "tile_edges": 3000, "tile_vertices": 3000,
                 "super_edges": 3000}


def _expected_super_edges(m, group=8192):
    """B's distinct edges per `group` consecutive faces of a one-object
    store, one entry per two faces sharing one (csrc/atiles.cu)."""
    total = 0
    for s0 in range(0, len(m), group):
        v = np.ascontiguousarray(m[s0:s0 + group]).reshape(-1, 3)
        _, vid = np.unique(v.view(np.dtype((np.void, 24))).ravel(), return_inverse=True)
        vid = vid.reshape(-1, 3)
        e = np.stack([np.sort(np.stack([vid[:, k], vid[:, (k + 1) % 3]], 1), 1) for k in range(3)], 1).reshape(-1, 2)
        _, cnt = np.unique(e, axis=0, return_counts=True)
        total += int(np.sum((cnt + 1) // 2))
    return total


def _expected_counts(m, obj_faces, tiles_per_group=256):
    """Numpy restatement of the A-side lists (csrc/atiles.cu): per super-tile
    (256 tiles of 128 faces of one object) the distinct edges, one entry per
    two faces sharing one; the distinct vertices, one entry per two of the
    tiles having one. Meshes here have no degenerate faces."""
    edges = verts = 0
    f0 = 0
    for nf in obj_faces:
        for s0 in range(0, nf, 128 * tiles_per_group):
            s1 = min(nf, s0 + 128 * tiles_per_group)
            v = np.ascontiguousarray(m[f0 + s0:f0 + s1]).reshape(-1, 3)
            _, vid = np.unique(v.view(np.dtype((np.void, 24))).ravel(), return_inverse=True)
            vid = vid.reshape(-1, 3)
            tile = (np.arange(s1 - s0) // 128)
            e = np.stack([np.sort(np.stack([vid[:, k], vid[:, (k + 1) % 3]], 1), 1) for k in range(3)], 1).reshape(-1, 2)
            _, cnt = np.unique(e, axis=0, return_counts=True)
            edges += int(np.sum((cnt + 1) // 2))
            vt = np.unique(np.stack([vid.ravel(), np.repeat(tile, 3)], 1), axis=0)
            _, tcnt = np.unique(vt[:, 0], return_counts=True)
            verts += int(np.sum((tcnt + 1) // 2))
        f0 += nf
    return edges, verts


def test_super_tile_counts_match_restatement():
    terrain = T.terrain(256, 160, 20.0, 7)          # 81,920 faces: rows of 512 faces (4 tiles)
    sphere = T.unit_sphere(100_000)                 # 81,920 faces, subdivision order
    for m in (terrain, sphere):
        c = T.Mesh(m).feature_counts()
        assert (c["tile_edges"], c["tile_vertices"]) == _expected_counts(m, [len(m)])
        assert c["super_edges"] == _expected_super_edges(m)
    recs = [T.unit_sphere(1000) + 3 * k for k in range(5)]
    tab = np.ascontiguousarray(np.concatenate(recs))
    off = np.arange(6, dtype=np.uint64) * len(recs[0])
    c = T.Table(tab, off).feature_counts()
    assert (c["tile_edges"], c["tile_vertices"]) == _expected_counts(tab, [len(r) for r in recs])


def test_row_selections_cutting_super_tiles():
    """A terrain of 327,680 faces (160 rows of 2,048 faces, 16 tiles per row:
    its super-tiles of 256 tiles are 16 rows, and an edge's two tiles are up
    to 16 tiles apart) against a small body: selections that start and end
    inside super-tiles read their tiles' entries plus the span before them,
    and must give the oracle's answer; so must the two-way shard split."""
    a = T.terrain(1024, 160, 20.0, 3)
    b = np.ascontiguousarray(T.ore_body(2000) * 0.05 + np.tile([500.0, 40.0, -30.0], 3))
    ma, mb = T.Mesh(a), T.Mesh(b)
    for r0, r1 in [(33_000, 70_001), (32_768, 65_536), (100, 40_000), (200_000, 327_680), (65_535, 65_537)]:
        r = T.mesh_mesh_distance(ma, mb, rows=(r0, r1))
        d, p, found, *_ = O.mesh_mesh_distance(a, b, rows=(r0, r1, 1))
        assert found and bits(r.distance) == bits(d) and r.pair_index == p, (r0, r1, r, d, p)
