"""Cost of the per-store builds on the e2e path: a fresh A store of 65,536
terrain rows each iteration against a resident ore body B: first call
(builds A's super-tile lists) vs a second call on the same stores."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1808_09571_b200 as T
T.init(0)
A = T.terrain(1024, 512, 20.0, 42)
B = T.Mesh(T.ore_body(1_000_000))
T.mesh_mesh_distance(T.Mesh(A[:8192]), B)  # B's feature blocks
pA = torch.from_numpy(A).pin_memory().numpy()
for it in range(4):
    r0 = it * 65536
    t0 = time.perf_counter()
    a = T.Mesh(pA[r0:r0 + 65536]); t1 = time.perf_counter()
    T.mesh_mesh_distance(a, B); t2 = time.perf_counter(); s1 = T.last_stats()
    T.mesh_mesh_distance(a, B); t3 = time.perf_counter(); s2 = T.last_stats()
    a.free()
    print(f"upload {1e3*(t1-t0):.1f} ms  first call {1e3*(t2-t1):.1f} (filter {s1['ms_filter']:.1f})  "
          f"second {1e3*(t3-t2):.1f} (filter {s2['ms_filter']:.1f})", flush=True)
