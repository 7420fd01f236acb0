"""tests/exact_tt.py (the exact rational checker the bound tests use) agrees
with the reference composition where the reference is well conditioned."""
import numpy as np
import pytest

import exact_tt as ET
import oracle as O


@pytest.mark.skipif(O.REF is None, reason="oracle/_ref not built")
def test_exact_checker_matches_reference_on_plain_pairs():
    rng = np.random.default_rng(3)
    a = rng.uniform(-1, 1, (60, 9))
    b = rng.uniform(-1, 1, (60, 9)) * 0.5 + rng.uniform(-1.5, 1.5, (60, 1)).repeat(9, 1)
    ref = O.ref_pairs_distance(a, b)[:, 0]
    for k in range(len(a)):
        true = float(ET.tri_tri_distance2(a[k], b[k])) ** 0.5
        assert abs(true - ref[k]) <= 1e-12 * max(1.0, ref[k]), (k, true, ref[k])
    # a crossing pair and a touching one
    t = np.array([0, 0, 0, 1, 0, 0, 0, 1, 0.0])
    assert ET.tri_tri_distance2(t, np.array([0.2, 0.2, -1, 0.3, 0.2, 1, 0.2, 0.3, 1.0])) == 0
    assert ET.tri_tri_distance2(t, t + np.array([0, 0, 2.0] * 3)) == 4
