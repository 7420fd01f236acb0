"""Time the pieces of the one-shot query path (host arrays in, results out)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1808_09571_b200 as T
T.init(0)
d = torch.from_numpy(T.drills(5_000_000, 42)).pin_memory().numpy()
ore = T.ore_body(500)
m = T.Mesh(ore)
for it in range(3):
    t0 = time.perf_counter(); q = T.Queries(d); t1 = time.perf_counter()
    r = T.queries_mesh_distance(q, m); t2 = time.perf_counter()
    q.free(); t3 = time.perf_counter()
    r2 = T.segments_mesh_distance(d, m); t4 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.1f} ms  eval {1e3*(t2-t1):.1f} ms  free {1e3*(t3-t2):.1f} ms  one-shot {1e3*(t4-t3):.1f} ms", T.last_stats()['ms_total'])
