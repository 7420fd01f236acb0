"""Device group (include/tindb_b200.h tdb_group_*): one process driving
several devices, A rows / table objects split over the members, one MIN
all-reduce. Results must equal the single-device call bit-for-bit (and so
the reference's, tests/test_gpu_parity.py).

The box the GPU tests run on has one B200: the NCCL path runs as a
one-member group; 2-8 member groups share device 0 under
TDB_GROUP_SHARED_DEVICES=1 (NCCL refuses duplicate devices, so their MIN
reductions go through host memory) to exercise the shard cuts and the
lexicographic reduction."""
import os

import numpy as np
import pytest

import oracle as O
import paper_1808_09571_b200 as T
from conftest import bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def device():
    T.init(0)
    os.environ["TDB_GROUP_SHARED_DEVICES"] = "1"
    yield
    os.environ.pop("TDB_GROUP_SHARED_DEVICES", None)


def same_dist(r, s):
    assert bits(r.distance) == bits(s.distance)
    assert r.pair_index == s.pair_index
    if s.pair_index is not None:
        assert np.array_equal(bits(np.array(r.closest_on_a)), bits(np.array(s.closest_on_a)))
        assert np.array_equal(bits(np.array(r.closest_on_b)), bits(np.array(s.closest_on_b)))


@pytest.mark.parametrize("members", [[0], [0, 0], [0, 0, 0], [0] * 8])
def test_group_mesh_mesh_matches_single_device(golden_meshes, members):
    g = T.Group(members)
    assert len(g) == len(members)
    for name, c in golden_meshes.items():
        ga, gb = g.mesh(c["a"]), g.mesh(c["b"])
        r = g.mesh_mesh_distance(ga, gb)
        assert bits(r.distance) == bits(c["dist"]), name
        assert (r.pair_index if r.pair_index is not None else O.U64_MAX) == int(c["pair"]), name
        if r.pair_index is not None:
            assert np.array_equal(bits(np.array(r.closest_on_a)), bits(c["on_a"])), name
        h = g.mesh_mesh_intersects(ga, gb)
        assert h.hit == bool(c["hit"]), name
        assert (h.pair_index if h.hit else O.U64_MAX) == int(c["hit_pair"]), name


def test_group_winner_in_late_shard_and_ties():
    """The minimum sits in the last member's rows; a translated copy makes
    an exact tie across shards (lowest pair must win)."""
    s = T.unit_sphere(10_000)                     # 8,192 faces
    b = T.translate(s, 2.5, 0, 0)                 # answer exactly 0.5
    a2 = np.concatenate([T.translate(s, 0, 0, 50.0), s])  # winner rows in the second half
    a3 = np.concatenate([s, s])                   # the same minimum in both halves: tie
    for members in ([0, 0], [0, 0, 0, 0]):
        g = T.Group(members)
        gb = g.mesh(b)
        for a in (a2, a3):
            same_dist(g.mesh_mesh_distance(g.mesh(a), gb), T.mesh_mesh_distance(a, b))
        c = T.translate(s, 0.5, 0, 0)
        gh = g.mesh_mesh_intersects(g.mesh(a2), g.mesh(c))
        h = T.mesh_mesh_intersects(a2, c)
        assert gh.hit == h.hit and gh.pair_index == h.pair_index
        st = [g.last_stats(m) for m in range(len(members))]
        assert sum(x["pairs"] for x in st) == len(a2) * len(c)


def test_group_table_matches_single_device(golden_table):
    t = golden_table
    for members in ([0], [0, 0, 0], [0] * 8):
        g = T.Group(members)
        gt, gl = g.table(t["table"], t["offsets"]), g.mesh(t["query"])
        d, dp = g.table_eval(T.OP_DISTANCE, gt, gl)
        assert np.array_equal(bits(d), bits(t["dist"])) and np.array_equal(dp, t["dist_pair"])
        h, hp = g.table_eval(T.OP_INTERSECTS, gt, gl)
        assert np.array_equal(h, t["hit"].astype(bool)) and np.array_equal(hp, t["hit_pair"])


def test_group_rejects_bad_devices(monkeypatch):
    with pytest.raises(ValueError):
        T.Group([T.device_count()])
    monkeypatch.setenv("TDB_GROUP_SHARED_DEVICES", "0")
    with pytest.raises(ValueError):
        T.Group([0, 0])


def test_group_intersects_shared_early_exit_keeps_lowest_hit():
    """Members share one lowest-hit word (intersects early exit across
    devices): a hit found first by a member with higher rows must not stop
    a member with lower rows from finding its lower hit."""
    s = T.unit_sphere(10_000)
    c = T.translate(s, 0.5, 0, 0)                       # hits
    far = T.translate(s, 0, 0, 50.0)                    # no hits
    for a in (np.concatenate([s, far, far, s]), np.concatenate([far, far, far, s]), np.concatenate([s, s, s, s])):
        h = T.mesh_mesh_intersects(a, c)
        for members in ([0], [0, 0], [0, 0, 0, 0], [0] * 8):
            g = T.Group(members)
            gh = g.mesh_mesh_intersects(g.mesh(a), g.mesh(c))
            assert gh.hit == h.hit and gh.pair_index == h.pair_index, members


def test_group_empty_and_single_face():
    s = T.unit_sphere(80)
    empty = np.zeros((0, 9))
    for members in ([0], [0, 0, 0]):
        g = T.Group(members)
        r = g.mesh_mesh_distance(g.mesh(empty), g.mesh(s))
        assert r.pair_index is None and r.distance == float("inf")
        assert not g.mesh_mesh_intersects(g.mesh(s), g.mesh(empty)).hit
        one = s[:1]
        same_dist(g.mesh_mesh_distance(g.mesh(one), g.mesh(T.translate(s, 3, 0, 0))),
                  T.mesh_mesh_distance(one, T.translate(s, 3, 0, 0)))
