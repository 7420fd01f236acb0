"""One small call of each kind (after a warm-up), for an ncu launch list."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1808_09571_b200 as T
T.init(0)
s = T.unit_sphere(1000)
a, b = T.Mesh(s), T.Mesh(T.translate(s, 2.5, 0, 0))
one = T.Mesh(s[:1])
seg = np.array([[0, 0, 2, 0, 0, 3.0]])
for rep in range(2):
    T.mesh_mesh_distance(one, one)
    T.mesh_mesh_distance(a, b)
    T.segments_mesh_distance(seg, a)
