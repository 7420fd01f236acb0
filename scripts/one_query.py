"""One resident drill-query call (profiling helper).
usage: python scripts/one_query.py {distance|intersects} N_DRILLS FACE_TARGET"""
import sys
sys.path.insert(0, '.')
import paper_1808_09571_b200 as T
op, n, ft = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
T.init(0)
q, ore = T.Queries(T.drills(n, 42)), T.Mesh(T.ore_body(ft))
r = T.queries_mesh_distance(q, ore) if op == "distance" else T.queries_mesh_intersects(q, ore)
print(T.last_stats())
