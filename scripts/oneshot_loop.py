"""Wall time of repeated one-shot tdb_distance_host calls on the C2 batch
(the bench's e2e step): upload A rows + B, evaluate, free."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1808_09571_b200 as T
T.init(0)
A = T.terrain(1024, 512, 20.0, 42); B = T.ore_body(1_000_000)
pA, pB = torch.from_numpy(A).pin_memory().numpy(), torch.from_numpy(B).pin_memory().numpy()
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8):
    r0 = (it % 16) * 65536
    t0 = time.perf_counter()
    r = T.distance_host(pA[r0:r0 + 65536], pB)
    t1 = time.perf_counter()
    s = T.last_stats()
    print(f"one-shot {1e3*(t1-t0):.1f} ms (filter {s['ms_filter']:.1f}, total {s['ms_total']:.1f})", flush=True)
