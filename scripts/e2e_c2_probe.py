"""Break down the C2 e2e step (one-shot tdb_distance_host) against the resident step."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1808_09571_b200 as T
T.init(0)
A = T.terrain(1024, 512, 20.0, 42); B = T.ore_body(1_000_000)
pA, pB = torch.from_numpy(A).pin_memory().numpy(), torch.from_numpy(B).pin_memory().numpy()
dA, dB = T.Mesh(A), T.Mesh(B)
R = 65536
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = T.mesh_mesh_distance(dA, dB, rows=(it * R, (it + 1) * R)); t1 = time.perf_counter()
    s1 = T.last_stats()
    a = T.Mesh(pA[it * R:(it + 1) * R]); t2 = time.perf_counter()
    b = T.Mesh(pB); t3 = time.perf_counter()
    r2 = T.mesh_mesh_distance(a, b); t4 = time.perf_counter()
    s2 = T.last_stats()
    a.free(); b.free(); t5 = time.perf_counter()
    r3 = T.distance_host(pA[it * R:(it + 1) * R], pB); t6 = time.perf_counter()
    s3 = T.last_stats()
    print(f"resident {1e3*(t1-t0):.1f} ms (filter {s1['ms_filter']:.1f} total {s1['ms_total']:.1f} items {s1.get('items')})")
    print(f"  upload A {1e3*(t2-t1):.1f}  upload B {1e3*(t3-t2):.1f}  eval {1e3*(t4-t3):.1f} (filter {s2['ms_filter']:.1f} total {s2['ms_total']:.1f})  free {1e3*(t5-t4):.1f}")
    print(f"  one-shot {1e3*(t6-t5):.1f} (filter {s3['ms_filter']:.1f} total {s3['ms_total']:.1f})")
    print("  ", {k: (s1[k], s2[k]) for k in s1 if s1[k] != s2[k]})
for it in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r3 = T.distance_host(pA[it * R:(it + 1) * R], pB); t1 = time.perf_counter()
    print(f"one-shot {1e3*(t1-t0):.1f}", flush=True)
