"""Repeated host->device store builds of the C2 ore body (pinned), each with
a distance call (feature blocks) and a free: per-iteration upload / call time.
usage: python scripts/upload_loop.py [iters]"""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1808_09571_b200 as T
T.init(0)
B = T.ore_body(1_000_000)
A = T.terrain(1024, 512, 20.0, 42)[:8192]
pB = torch.from_numpy(B).pin_memory().numpy()
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8):
    t0 = time.perf_counter()
    b = T.Mesh(pB); t1 = time.perf_counter()
    a = T.Mesh(A)
    r = T.mesh_mesh_distance(a, b); t2 = time.perf_counter()
    a.free(); b.free(); t3 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.1f} ms  call {1e3*(t2-t1):.1f} ms (filter {T.last_stats()['ms_filter']:.1f})  free {1e3*(t3-t2):.1f} ms", flush=True)
