"""Small-call crossover: wall time per mesh x mesh distance / intersects call
for A rows x 1,280 B faces, in whichever path TDB_DIRECT_PAIRS selects
(run once with TDB_DIRECT_PAIRS=0 and once with a large value)."""
import json, os, sys, time
sys.path.insert(0, '.')
import paper_1808_09571_b200 as T
T.init(0)
s = T.unit_sphere(1000)
b = T.Mesh(T.translate(s, 2.5, 0, 0))
for rows in (16, 32, 64, 128, 256, 512):
    a = T.Mesh(s[:rows])
    for op, f in (("distance", T.mesh_mesh_distance), ("intersects", T.mesh_mesh_intersects)):
        for _ in range(20):
            f(a, b)
        t0 = time.perf_counter()
        for _ in range(200):
            f(a, b)
        us = (time.perf_counter() - t0) / 200 * 1e6
        print(json.dumps({"direct_pairs": os.environ.get("TDB_DIRECT_PAIRS"), "op": op, "pairs": rows * len(s),
                          "us_per_call": round(us, 1), "kernels": T.last_stats()["kernels"]}), flush=True)
