"""First-contact probe: FP64 peak, C2 distance at three row counts, C3 intersects (resident meshes)."""
import time, sys, json
sys.path.insert(0, '.')
import numpy as np
import paper_1808_09571_b200 as T
T.init(0)
tf, ms = T.fp64_peak(); print("fp64 peak TF", tf, "ms", ms)
ter = T.terrain(); ore = T.ore_body(1000000)
print(ter.shape, ore.shape)
A = T.Mesh(ter); B = T.Mesh(ore)
for rows in [(0, 1024), (0, 8192), (0, 65536)]:
    t0 = time.time(); r = T.mesh_mesh_distance(A, B, rows=rows); t1 = time.time()
    st = T.last_stats()
    print(rows, r.distance, r.pair_index, "wall", t1-t0, st, "pairs/s filter", st['pairs']/(st['ms_filter']*1e-3))
s = T.unit_sphere(1000000)
S = T.Mesh(s); S9 = T.Mesh(s*0.9)
t0=time.time(); h = T.mesh_mesh_intersects(S, S9, rows=(0, 65536)); t1=time.time()
st = T.last_stats(); print("intersects", h, t1-t0, st, "pairs/s", st['pairs']/(st['ms_filter']*1e-3))
