import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_1808_09571_b200 as T, oracle as O
import test_gpu_fuzz as F
T.init(0)
bad = 0
for seed in range(3):
    rng = np.random.default_rng(1000 + seed)
    for c in range(25):
        st0 = rng.bit_generator.state
        kind = np.random.default_rng().integers(0, 1)
        a, b = F._case(rng)
        r = T.mesh_mesh_distance(a, b)
        st = T.last_stats()
        d, p, found, wa, wb = O.mesh_mesh_distance(a, b)
        if np.float64(r.distance).view(np.uint64) != np.float64(d).view(np.uint64):
            bad += 1
            ia, ib = T.Mesh(a).info(), T.Mesh(b).info()
            print("BAD seed", seed, "case", c, len(a), len(b), r.distance, r.pair_index, d, p, st)
            print("   degen", ia['degenerate'], ib['degenerate'], "aabb", ia['aabb'])
            np.savez(f"gpurun_out/fuzzbad_{seed}_{c}.npz", a=a, b=b)
print("bad", bad)
