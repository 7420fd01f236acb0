"""One resident-mesh call on the C2 meshes (profiling helper).
usage: python scripts/one_call.py {distance|intersects} ROWS"""
import sys
sys.path.insert(0, '.')
import paper_1808_09571_b200 as T
op, rows = sys.argv[1], int(sys.argv[2])
T.init(0)
if op == "distance":
    A, B = T.Mesh(T.terrain()), T.Mesh(T.ore_body(1_000_000))
    r = T.mesh_mesh_distance(A, B, rows=(0, rows))
else:
    s = T.unit_sphere(1_000_000)
    A, B = T.Mesh(s), T.Mesh(s * 0.9)
    r = T.mesh_mesh_intersects(A, B, rows=(0, rows))
print(r, T.last_stats())
