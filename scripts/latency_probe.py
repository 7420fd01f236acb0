"""Per-call latency of the C ABI for small inputs (the serving path), wall
time per call after warm-up. Prints one JSON object per call kind."""
import json
import sys
import time

sys.path.insert(0, '.')
import numpy as np

import paper_1808_09571_b200 as T

T.init(0)
s = T.unit_sphere(1000)
a, b = T.Mesh(s), T.Mesh(T.translate(s, 2.5, 0, 0))
one, one2 = T.Mesh(s[:1]), T.Mesh(T.translate(s[:1], 0, 0, 3.0))
small = T.Mesh(s[:64])
tab = T.Table(np.concatenate([T.translate(s, 3 * k, 0, 0) for k in range(16)]), np.arange(17, dtype=np.uint64) * len(s))
seg = np.array([[0, 0, 2, 0, 0, 3.0]])
pt = np.array([[0.1, 0.2, 1.5]])


def t(f, n=400):
    for _ in range(20):
        f()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    return (time.perf_counter() - t0) / n * 1e6


for name, f in [("distance 1x1", lambda: T.mesh_mesh_distance(one, one2)),
                ("intersects 1x1", lambda: T.mesh_mesh_intersects(one, one2)),
                ("distance 64x1280", lambda: T.mesh_mesh_distance(small, b)),
                ("segment query 1 x 1280 faces", lambda: T.segments_mesh_distance(seg, a)),
                ("point query 1 x 1280 faces", lambda: T.points_mesh_distance(pt, a)),
                ("segment intersects 1 x 1280", lambda: T.segments_mesh_intersects(seg, a)),
                ("distance 1280x1280", lambda: T.mesh_mesh_distance(a, b)),
                ("intersects 1280x1280", lambda: T.mesh_mesh_intersects(a, b)),
                ("table_eval 16 rec x 1280", lambda: T.table_eval(T.OP_DISTANCE, tab, b)),
                ("upload 1280 faces", lambda: T.Mesh(s).free())]:
    us = t(f)
    st = T.last_stats()
    print(json.dumps({"call": name, "us_per_call": round(us, 1), "device_us": round(st["ms_total"] * 1e3, 1),
                      "kernels": st["kernels"]}), flush=True)
