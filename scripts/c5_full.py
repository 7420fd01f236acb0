"""The whole C5 job (8,388,608^2 = 7.04e13 triangle pairs, ST_3DDistance) in one
C-ABI call on one B200, checked against the analytic answer (0.5) and the
AABB-pruned exact CPU oracle (lexicographic (distance, pair))."""
import json, sys, time
sys.path.insert(0, '.')
import numpy as np
import oracle as O
import paper_1808_09571_b200 as T
T.init(0)
s = T.unit_sphere(10_000_000)
b = T.translate(s, 2.5, 0.0, 0.0)
A, B = T.Mesh(s), T.Mesh(b)
t0 = time.perf_counter()
r = T.mesh_mesh_distance(A, B)
wall = time.perf_counter() - t0
st = T.last_stats()
d, p, found, *_ = O.mesh_mesh_distance_pruned(s, b, r.distance)
out = {"faces": len(s), "pairs": st["pairs"], "distance": r.distance, "pair": r.pair_index,
       "wall_s": wall, "ms_filter": st["ms_filter"], "pairs_per_s": st["pairs"] / (st["ms_filter"] * 1e-3),
       "oracle_distance": d, "oracle_pair": p, "match": bool(found and d == r.distance and p == r.pair_index),
       "analytic_0_5": r.distance == 0.5}
print(json.dumps(out))
json.dump(out, open("gpurun_out/c5_full.json", "w"), indent=1)
