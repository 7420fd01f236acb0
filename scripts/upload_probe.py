"""Time mesh upload (H2D + prep) and free for the C2 meshes from pinned memory."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1808_09571_b200 as T
T.init(0)
ore = torch.from_numpy(T.ore_body(1_000_000)).pin_memory().numpy()
ter = torch.from_numpy(T.terrain()).pin_memory().numpy()
for it in range(4):
    t0 = time.perf_counter(); m = T.Mesh(ore); t1 = time.perf_counter(); m.free(); t2 = time.perf_counter()
    a = T.Mesh(ter[:65536]); t3 = time.perf_counter(); a.free(); t4 = time.perf_counter()
    t5 = time.perf_counter(); r = T.distance_host(ter[:1024], ore); t6 = time.perf_counter()
    st = T.last_stats()
    print(f"ore upload {1e3*(t1-t0):.1f} free {1e3*(t2-t1):.1f} | batch upload {1e3*(t3-t2):.1f} free {1e3*(t4-t3):.1f} | one-shot 1024 rows {1e3*(t6-t5):.1f} ms (device {st['ms_total']:.1f})")
