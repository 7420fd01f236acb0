"""C1 distance call statistics (flagged items, candidates, timings)."""
import sys
sys.path.insert(0, '.')
import paper_1808_09571_b200 as T
T.init(0)
s = T.unit_sphere(10000)
a, b = T.Mesh(s), T.Mesh(T.translate(s, 2.5, 0, 0))
for _ in range(3):
    r = T.mesh_mesh_distance(a, b)
print(r.distance, T.last_stats())
