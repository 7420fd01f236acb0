"""ST_3DVolume timings (mesh_volume on the device, resident mesh) for the paper's 500-face ore and the
1.31M-face ore, next to the reference's own mesh_volume on one host thread."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import oracle as O
import paper_1808_09571_b200 as T
T.init(0)
for ft in (500, 1_000_000):
    ore = T.ore_body(ft)
    m = T.Mesh(ore)
    for _ in range(3):
        v = T.mesh_volume(m)
    t0 = time.perf_counter()
    for _ in range(20):
        v = T.mesh_volume(m)
    dt = (time.perf_counter() - t0) / 20
    st = T.last_stats()
    ref = getattr(O, "ref_mesh_volume", None)
    line = f"{len(ore)} faces: device {dt * 1e6:.1f} us/call (kernel {st['ms_total'] * 1e3:.1f} us), volume {v!r}"
    if ref is not None:
        t0 = time.perf_counter(); rv = ref(ore); rdt = time.perf_counter() - t0
        rv = rv[0] if isinstance(rv, tuple) else rv
        line += f"; reference {rdt * 1e3:.2f} ms, bit-equal {np.float64(rv).view(np.uint64) == np.float64(v).view(np.uint64)}"
    print(line)
