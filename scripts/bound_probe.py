"""Dump the worst filter-bound violations of tests/test_gpu_bounds.py inputs."""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
import paper_1808_09571_b200 as T
import test_gpu_bounds as G
T.init(0)
for seed in (11, 12):
    a, b = G.adversarial_pairs(seed, 1_000_000)
    ref = T.pairs_distance(a, b)
    d2 = T.pairs_filter(a, b)
    fin = np.isfinite(ref)
    idx = np.flatnonzero(fin)
    dt, r = np.sqrt(d2[fin]), ref[fin]
    A, B = a[fin].reshape(-1, 3, 3), b[fin].reshape(-1, 3, 3)
    edge = np.maximum(np.linalg.norm(A - np.roll(A, -1, 1), axis=2).max(1), np.linalg.norm(B - np.roll(B, -1, 1), axis=2).max(1))
    scale = np.maximum(np.abs(A).max((1, 2)), np.abs(B).max((1, 2)))
    tol = 1e-7 * edge + 1e-12 * scale + 1e-6 * r
    ratio = np.abs(dt - r) / tol
    bad = np.argsort(-ratio)[:50]
    k = 1_000_000 // 5
    print(seed, "violations:", (ratio > 1).sum(), "families:", np.bincount(idx[ratio > 1] // k, minlength=5), "max", ratio.max())
    np.savez(f"gpurun_out/bound_{seed}.npz", a=a[idx[bad]], b=b[idx[bad]], ref=r[bad], filt=dt[bad], ratio=ratio[bad], fam=idx[bad] // k,
             signed=(dt - r)[bad])
    neg = (dt - r) / tol
    print("  most negative (filter below ref):", neg.min(), " most positive:", neg.max())
