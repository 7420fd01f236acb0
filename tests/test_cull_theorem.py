"""The intersects culls against the reference's own noisy arithmetic
(DESIGN.md 4.3), on CPU: the reference (oracle/_ref) decides every pair of
the adversarial families in tests/adversarial.py, and

* the round-1 cull (one-way plane test, tau = 1e-10 D) is shown to drop
  reference hits there (the advisor's sliver finding, and the grazing
  near-parallel family), while
* the round-2 culls (tdb_internal.h kCullOne / kCullTwo / kApart with the
  per-face kappa) never drop one, even at the pair-level D (the tightest the
  device may use; the device's object-level D only widens the margins).
"""
import numpy as np
import pytest

import adversarial as AD
import oracle as O

pytestmark = pytest.mark.skipif(O.REF is None, reason="oracle/_ref not built")


def _families(seed, n=40_000):
    rng = np.random.default_rng(seed)
    for w in (1e-8, 1e-10, 1e-12, 1e-13):
        recs, lit = AD.sliver_literal(rng, n, w)
        yield f"sliver_literal w={w:g}", recs, np.repeat(lit, n, 0)
    recs, lit = AD.sliver_records(rng, n)
    yield "sliver_records", recs, np.repeat(lit, n, 0)
    for _ in range(2):
        recs, lit = AD.grazing_parallel(rng, n)
        yield "grazing_parallel", recs, np.repeat(lit, n, 0)


@pytest.mark.parametrize("seed", [1, 2])
def test_new_culls_never_drop_a_reference_hit(seed):
    old_misses = 0
    for name, a, b in _families(seed):
        ref = O.ref_pairs_intersects(a, b).astype(bool)
        new = AD.new_cull_separates(a, b)
        bad = np.flatnonzero(ref & new)
        assert len(bad) == 0, (name, len(bad), a[bad[:2]], b[bad[:2]])
        old_misses += int((ref & AD.old_cull_separates(a, b)).sum())
        print(f"{name}: {ref.sum()} reference hits, {new.sum()} culled")
    # the families do exercise the noise the round-1 cull ignored
    assert old_misses > 1000, old_misses


def test_segment_culls_never_drop_a_reference_hit():
    """Segment x face (q_hit / lt_hit): apart kApart D, t-rejection with
    (kCullTwo + kappa) D, D = the pair's box diagonal."""
    rng = np.random.default_rng(9)
    mesh, segs = AD.sliver_mesh_and_segments(rng, 400, 40_000)
    hit, face = O.ref_segments_mesh_intersects(segs, mesh)
    assert hit.sum() > 100
    hit = hit.astype(bool)
    # for each hit: the winning face must not be culled
    f = face[hit].astype(np.int64)
    s, t = segs[hit], mesh[f]
    P, Q = s[:, 0:3], s[:, 3:6]
    box_lo = np.minimum(np.minimum(P, Q), t.reshape(-1, 3, 3).min(1))
    box_hi = np.maximum(np.maximum(P, Q), t.reshape(-1, 3, 3).max(1))
    D = np.linalg.norm(box_hi - box_lo, axis=1)
    ab = 1e-13 * np.maximum(np.abs(s).max(1), np.abs(t).max(1))
    n, c = AD._plane(t)
    h0, h1 = (n * P).sum(1) - c, (n * Q).sum(1) - c
    tau = (1.01e-12 + AD.kappa(t)) * D + ab
    culled = ((h0 > tau) & (h1 > tau)) | ((h0 < -tau) & (h1 < -tau))
    gap = 5e-2 * D + ab
    T = t.reshape(-1, 3, 3)
    apart = ((T.min(1) > np.maximum(P, Q) + gap[:, None]) | (T.max(1) < np.minimum(P, Q) - gap[:, None])).any(1)
    assert not (culled | apart).any()
    # and the round-1 segment cull (tau = 1e-10 D) would have dropped some
    old_tau = 1e-10 * D + ab
    old = ((h0 > old_tau) & (h1 > old_tau)) | ((h0 < -old_tau) & (h1 < -old_tau))
    print(f"{hit.sum()} segment hits; round-1 cull drops {old.sum()}")
