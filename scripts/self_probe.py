"""Pathological exact-pass loads: a mesh against itself (every face ties at 0)
and against a nearly coincident copy."""
import sys, time
sys.path.insert(0, '.')
import paper_1808_09571_b200 as T
T.init(0)
for ft in (100_000, 1_000_000):
    s = T.unit_sphere(ft)
    for name, b in (("self", s), ("shift1e-9", T.translate(s, 1e-9, 0, 0))):
        A, B = T.Mesh(s), T.Mesh(b)
        t0 = time.perf_counter(); r = T.mesh_mesh_distance(A, B); dt = time.perf_counter() - t0
        st = T.last_stats()
        print(f"{len(s)} {name}: {dt*1e3:.1f} ms filter {st['ms_filter']:.1f} verify {st['ms_verify']:.1f} "
              f"flagged {st['items_flagged']}/{st['items']} cand {st['candidates']} rounds {st['rounds']} -> {r.distance} {r.pair_index}")
