"""World-size-2 gloo tests of the multi-rank host logic (shard.py) on CPU.

Each rank evaluates its row shard with the CPU oracle (standing in for its
GPU), then the ranks reduce with the same collectives bench.py uses over
NCCL; the reduced answer must equal the single-process answer bit-for-bit.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import oracle as O
from paper_1808_09571_b200 import shard


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def meshes():
    rng = np.random.default_rng(12)
    a = rng.uniform(-1, 1, (300, 9))
    b = rng.uniform(-1, 1, (170, 9)) * 0.6 + 0.9
    return a, b


def table():
    rng = np.random.default_rng(3)
    objs = [rng.uniform(-1, 1, (int(n), 9)) * 0.2 + rng.uniform(-2, 2, 3).repeat(3)[None, :]
            for n in rng.integers(0, 40, 13)]
    off = np.cumsum([0] + [len(o) for o in objs])
    return np.concatenate(objs), off, rng.uniform(-1, 1, (60, 9))


def worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b = meshes()
        r0, r1 = shard.row_shards(len(a), world)[rank]
        d, p, found, _, _ = O.mesh_mesh_distance(a, b, threads=1, rows=(r0, r1, 1))
        best = shard.combine_min(d, p if found else None)
        hit, hp = O.mesh_mesh_intersects(a, b * 1.0 - 0.45, threads=1, rows=(r0, r1, 1))
        lowest = shard.combine_hit(hp if hit else None)
        t, off, qm = table()
        o0, o1 = shard.object_shards(off, world)[rank]
        dd, pp = O.table_eval("distance", t[off[o0]:off[o1]], off[o0:o1 + 1] - off[o0], qm, threads=1)
        counts = [e - s for s, e in shard.object_shards(off, world)]
        allp = shard.gather_slices(pp, counts)
        alld = shard.gather_slices(dd, counts)
        # no rank holds a pair: bench.py passes U64_MAX, the shard API None
        nohit = (shard.combine_min(float("inf"), shard.U64_MAX), shard.combine_min(float("inf"), None),
                 shard.combine_hit(shard.U64_MAX), shard.combine_hit(None))
        # bench.py's own step -> rank plan, weak and strong, each step reduced
        steps = {}
        for strong in (False, True):
            wl = bench.MeshWorkload("t", "distance", "t", lambda gen: (a, b), 128)
            wl.build(None)
            n_steps = wl.n_batches if strong else -(-wl.n_batches // world)
            res = []
            for s_ in range(n_steps):
                lo, hi = wl.span(s_, rank, world, strong)
                if not strong and s_ * world + rank >= wl.n_batches:
                    lo, hi = 0, 0  # past the end of the job: this rank idles
                d_, p_, f_, _, _ = O.mesh_mesh_distance(a, b, threads=1, rows=(lo, hi, 1))
                res.append(shard.combine_min(d_, p_ if f_ else shard.U64_MAX))
            steps[strong] = shard.lexmin(res)
        if rank == 0:
            q.put((best, lowest, alld, allp, nohit, steps))
    finally:
        dist.destroy_process_group()


def test_row_and_object_shards_cover_exactly():
    for n in [0, 1, 127, 128, 129, 1000, 1310720]:
        for w in [1, 2, 3, 8]:
            sh = shard.row_shards(n, w)
            assert sh[0][0] == 0 and sh[-1][1] == n
            assert all(sh[i][1] == sh[i + 1][0] for i in range(w - 1))
            assert all(s % shard.TILE == 0 for s, _ in sh)
    off = [0, 5, 5, 100, 101, 400, 402]
    for w in [1, 2, 4, 6, 9]:
        sh = shard.object_shards(off, w)
        assert sh[0][0] == 0 and sh[-1][1] == len(off) - 1
        assert all(sh[i][1] == sh[i + 1][0] for i in range(w - 1))


def test_lexmin_ties_keep_lowest_pair():
    assert shard.lexmin([(0.5, 9), (0.5, 3), (0.7, 1)]) == (0.5, 3)
    assert shard.lexmin([]) == (float("inf"), shard.U64_MAX)


@pytest.mark.timeout(180)
def test_two_rank_gloo_reduction_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    best, lowest, alld, allp, nohit, steps = q.get(timeout=170)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    a, b = meshes()
    d, p, found, _, _ = O.mesh_mesh_distance(a, b, threads=2)
    assert np.float64(best[0]).view(np.uint64) == np.float64(d).view(np.uint64) and best[1] == p
    hit, hp = O.mesh_mesh_intersects(a, b - 0.45, threads=2)
    assert lowest == (hp if hit else None)
    t, off, qm = table()
    dd, pp = O.table_eval("distance", t, off, qm, threads=2)
    assert np.array_equal(alld.view(np.uint64), dd.view(np.uint64)) and np.array_equal(allp, pp)
    inf = float("inf")
    assert nohit == ((inf, shard.U64_MAX), (inf, shard.U64_MAX), None, None)
    for strong in (False, True):
        assert np.float64(steps[strong][0]).view(np.uint64) == np.float64(d).view(np.uint64), strong
        assert steps[strong][1] == p, strong
