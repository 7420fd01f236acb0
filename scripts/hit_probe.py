"""One intersects call of 131,072 rows on C3 (sphere vs 0.9x copy) and on
the C3 stress pair (0.999x copy rotated 0.37 rad): pairs/s of hit_kernel."""
import sys
sys.path.insert(0, '.')
import bench
import paper_1808_09571_b200 as T
T.init(0)
for name in ("c3", "c3s"):
    wl = bench.workload(name, None, 0)
    wl.build(bench.ProductGen())
    a, b = T.Mesh(wl.A), T.Mesh(wl.B)
    for _ in range(2):
        h = T.mesh_mesh_intersects(a, b, rows=(0, 131072))
    s = T.last_stats()
    print(f"{name}: hit {h.hit}  {s['pairs'] / (s['ms_filter'] * 1e-3):.4g} pairs/s  ({s['ms_filter']:.2f} ms, exact pairs {s['exact_pairs']})")
