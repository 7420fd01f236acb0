"""Per-call latency floor of the C ABI for small inputs (serving path)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_1808_09571_b200 as T
T.init(0)
s = T.unit_sphere(1000)
a, b = T.Mesh(s), T.Mesh(T.translate(s, 2.5, 0, 0))
one = T.Mesh(s[:1])
tab = T.Table(np.concatenate([T.translate(s, 3 * k, 0, 0) for k in range(16)]), np.arange(17, dtype=np.uint64) * len(s))
seg = np.array([[0, 0, 2, 0, 0, 3.0]])
def t(f, n=200):
    for _ in range(5): f()
    t0 = time.perf_counter()
    for _ in range(n): f()
    return (time.perf_counter() - t0) / n * 1e6
for name, f in [("mesh_mesh_distance 1280x1280", lambda: T.mesh_mesh_distance(a, b)),
                ("mesh_mesh_distance 1x1", lambda: T.mesh_mesh_distance(one, one)),
                ("mesh_mesh_intersects 1280x1280", lambda: T.mesh_mesh_intersects(a, b)),
                ("table_eval 16 rec x 1280", lambda: T.table_eval(T.OP_DISTANCE, tab, b)),
                ("segments_mesh_distance 1 seg", lambda: T.segments_mesh_distance(seg, a)),
                ("upload 1280 faces", lambda: T.Mesh(s).free())]:
    us = t(f)
    st = T.last_stats()
    print(f"{name:34s} {us:8.1f} us/call  (device {st['ms_total']*1e3:.1f} us, kernels {st['kernels']})")
