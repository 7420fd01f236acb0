"""Concurrent callers (the reference server's contract: plan_and_execute →
run_batch from one thread per connection, /root/reference/proj/src/
pg_server.cpp:231,496; kernels are reentrant).

8 host threads issue mixed C-ABI calls on shared device handles — mesh x mesh
distance and intersects, table_eval both ops, segment / point queries, a
literal over a mesh column, one-shot host-buffer calls, uploads and frees of
their own meshes — each call on its own pooled stream (capi.cu). Every
answer must be bit-identical to the single-thread answer. ctypes releases
the GIL for the duration of each call, so the calls really overlap.
"""
import os
import threading

import numpy as np
import pytest

import paper_1808_09571_b200 as T
from conftest import bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def device():
    T.init(0)
    yield


def _work():
    s = T.unit_sphere(10000)
    rng = np.random.default_rng(1)
    objs = [T.translate(T.unit_sphere(1000) * rng.uniform(0.2, 1.0), *rng.uniform(-3, 3, 3)) for _ in range(24)]
    off = np.cumsum([0] + [len(o) for o in objs]).astype(np.uint64)
    segs = np.concatenate([rng.uniform(-2, 2, (500, 3)), rng.uniform(-2, 2, (500, 3))], 1)
    return {
        "A": T.Mesh(s), "B": T.Mesh(T.translate(s, 2.5, 0.1, 0.0)), "C": T.Mesh(T.translate(s, 0.5, 0.0, 0.0)),
        "tab": T.Table(np.concatenate(objs), off), "segs": segs, "s": s,
        "lit": np.array([0.1, 0.2, -0.3, 1.5, -0.4, 0.9]),
    }


def _calls(w):
    """name -> zero-argument callable returning comparable numpy arrays."""
    A, B, C, tab = w["A"], w["B"], w["C"], w["tab"]
    return {
        "dist": lambda: np.array([T.mesh_mesh_distance(A, B).distance, T.mesh_mesh_distance(A, B).pair_index]),
        "hit": lambda: np.array([T.mesh_mesh_intersects(A, C).pair_index], np.uint64),
        "tab_d": lambda: np.concatenate([x.view(np.uint64) for x in T.table_eval(T.OP_DISTANCE, tab, A)]),
        "tab_h": lambda: np.concatenate([x.astype(np.uint64) for x in T.table_eval(T.OP_INTERSECTS, tab, C)]),
        "seg_d": lambda: np.concatenate([x.view(np.uint64) for x in T.segments_mesh_distance(w["segs"], A)]),
        "seg_h": lambda: np.concatenate([x.astype(np.uint64) for x in T.segments_mesh_intersects(w["segs"], A)]),
        "pt_d": lambda: np.concatenate([x.view(np.uint64) for x in T.points_mesh_distance(w["segs"][:, :3], B)]),
        "lit": lambda: np.concatenate([x.view(np.uint64) for x in T.literal_table_eval(T.OP_DISTANCE, w["lit"], tab)]),
        "own": lambda: np.array([T.mesh_mesh_distance(T.Mesh(w["s"][:2000]), B).distance]),  # upload + free
        "host": lambda: np.array([T.distance_host(w["s"][:3000], w["s"][:1000] + 3.0).distance]),
    }


def test_eight_threads_mixed_calls_bit_identical():
    w = _work()
    calls = _calls(w)
    want = {k: f() for k, f in calls.items()}
    names = list(calls)
    errors, got = [], {}

    def worker(t):
        try:
            order = np.random.default_rng(t).permutation(len(names) * 3) % len(names)
            for i in order:
                k = names[i]
                r = calls[k]()
                if not np.array_equal(np.asarray(r).view(np.uint64) if r.dtype == np.float64 else r,
                                      np.asarray(want[k]).view(np.uint64) if want[k].dtype == np.float64
                                      else want[k]):
                    errors.append((t, k))
            got[t] = True
        except Exception as e:  # pragma: no cover - reported below
            errors.append((t, repr(e)))

    th = [threading.Thread(target=worker, args=(t,)) for t in range(8)]
    for x in th:
        x.start()
    for x in th:
        x.join(float(os.environ.get("TDB_TEST_JOIN_S", "600")))  # raise under compute-sanitizer
    assert not errors, errors[:10]
    assert len(got) == 8
    # each thread keeps its own last-call stats and error state
    T.mesh_mesh_distance(w["A"], w["B"])
    assert T.last_stats()["pairs"] == len(w["s"]) ** 2
