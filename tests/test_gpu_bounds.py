"""The two engineering bounds of the fast paths, stressed at scale on the
device (DESIGN.md section 7 names them as validated, not proven):

* the distance filter's error |d~ - d| <= eta (+ the 2^-20 high-word
  truncation), where d is the reference composition (tdb_pairs_distance,
  bit-identical to the reference, tests/test_gpu_parity.py) — the invariant
  the exact pass's band relies on (distance.cu, tdb_internal.h);
* the intersects plane cull's margin tau: a table of one-face records
  against a one-face literal runs the production hit_kernel (cull, then the
  exact predicate for survivors); every boolean must equal the exact
  predicate evaluated on every pair (tdb_pairs_intersects).

Inputs are seeded adversarial families: near-parallel edge pairs at graded
angles and separations, near-coplanar and grazing placements, slivers and
needles (aspect ratios to 1e6), near-contact clusters, each under random
rigid motions at scales 1e-3..1e3 and offsets up to 1e6.
"""
import numpy as np
import pytest

import exact_tt as ET
import oracle as O
import paper_1808_09571_b200 as T

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def device():
    T.init(0)
    yield


def _rots(rng, n):
    q, r = np.linalg.qr(rng.normal(size=(n, 3, 3)))
    return q * np.sign(np.diagonal(r, axis1=1, axis2=2))[:, None, :]


def _place(tri, R, t, s):
    v = tri.reshape(-1, 3, 3)
    return (np.einsum("nij,nkj->nki", R, v) * s[:, None, None] + t[:, None, :]).reshape(-1, 9)


def adversarial_pairs(seed, n):
    rng = np.random.default_rng(seed)
    k = n // 6
    out_a, out_b = [], []
    # 1. near-parallel edge pairs: a's edge v0v1 on the x axis, b's edge tilted by ang, lifted by sep
    ang = 10.0 ** rng.uniform(-16, -1, k) * rng.choice([-1, 1], k)
    sep = np.where(rng.random(k) < 0.2, 0.0, 10.0 ** rng.uniform(-14, 0, k))
    x0 = rng.uniform(-0.5, 1.5, k)
    a = np.tile([0, 0, 0, 1, 0, 0, 0.5, -1, -0.3], (k, 1)).astype(float)
    a[:, 6:9] += rng.normal(scale=0.3, size=(k, 3))
    b = np.stack([x0, sep, np.zeros(k), x0 + 1, sep + ang, np.zeros(k),
                  x0 + rng.uniform(-1, 1, k), sep + rng.uniform(0.2, 1, k), rng.uniform(-0.5, 0.5, k)], 1)
    out_a.append(a), out_b.append(b)
    # 2. near-coplanar: b in a's plane up to a tilt, overlapping or grazing
    a = rng.uniform(-1, 1, (k, 9))
    a[:, 2::3] = 0.0
    b = rng.uniform(-1, 1, (k, 9))
    b[:, 2::3] = 10.0 ** rng.uniform(-15, -2, (k, 1)) * rng.normal(size=(k, 3))
    out_a.append(a), out_b.append(b)
    # 3. slivers and needles (aspect ratio up to 1e6) near a random triangle
    a = rng.uniform(-1, 1, (k, 9))
    p = rng.uniform(-1, 1, (k, 3))
    d = rng.normal(size=(k, 3))
    w = 10.0 ** rng.uniform(-6, 0, (k, 1)) * rng.normal(size=(k, 3))
    b = np.concatenate([p, p + d, p + 0.5 * d + w], 1)
    out_a.append(a), out_b.append(b)
    # 4. vertex / edge contact: b's vertex placed at a point of a (edge or interior) plus a tiny offset
    a = rng.uniform(-1, 1, (k, 9))
    u, v = rng.random(k), rng.random(k)
    on_edge = rng.random(k) < 0.5
    v = np.where(on_edge, 0.0, v * (1 - u))
    q = a[:, 0:3] + u[:, None] * (a[:, 3:6] - a[:, 0:3]) + v[:, None] * (a[:, 6:9] - a[:, 0:3])
    q += 10.0 ** rng.uniform(-15, -3, (k, 1)) * rng.normal(size=(k, 3))
    b = np.concatenate([q, q + rng.normal(size=(k, 3)), q + rng.normal(size=(k, 3))], 1)
    out_a.append(a), out_b.append(b)
    # 5. near-contact clusters of random triangles
    m = n - 5 * k
    a = rng.uniform(-1, 1, (m, 9))
    b = rng.uniform(-1, 1, (m, 9)) * 0.3 + np.tile(a.reshape(m, 3, 3).mean(1) + rng.normal(scale=0.05, size=(m, 3)), 3)
    out_a.append(a), out_b.append(b)
    # 6. sliver interiors: a vertex of a hovering 1e-15..1e-3 over the inside of a
    #    sliver b (width 1e-13..1e-4: conditioning K = |e0||e1|/|N| up to 1e13),
    #    its projection a fraction of the width from the long edges
    w = 10.0 ** rng.uniform(-13, -4, k)
    L = rng.uniform(0.3, 2.0, k)
    b = np.stack([np.zeros(k), np.zeros(k), np.zeros(k), L, np.zeros(k), np.zeros(k), 0.5 * L, w, np.zeros(k)], 1)
    x = rng.uniform(0.05, 0.95, k) * L
    y = rng.uniform(0.0, 1.0, k) * w * (1 - np.abs(2 * x / L - 1))
    z = 10.0 ** rng.uniform(-15, -3, k) * rng.choice([-1, 1], k)
    p = np.stack([x, y, z], 1)
    a = np.concatenate([p, p + rng.normal(size=(k, 3)) + [0, 0, 2.0], p + rng.normal(size=(k, 3)) + [0, 0, 2.0]], 1)
    a[:, 5] = np.abs(a[:, 5]) * np.sign(z)  # the other two vertices on the same side as the hovering one
    a[:, 8] = np.abs(a[:, 8]) * np.sign(z)
    out_a.append(a), out_b.append(b)
    a, b = np.concatenate(out_a), np.concatenate(out_b)
    # random rigid motion, scale, offset (shared by both triangles of a pair)
    N = len(a)
    R = _rots(rng, N)
    s = 10.0 ** rng.integers(-3, 4, N).astype(float)
    t = np.where(rng.random((N, 1)) < 0.3, rng.uniform(-1, 1, (N, 3)) * 1e6, rng.uniform(-3, 3, (N, 3)))
    return _place(a, R, t, s), _place(b, R, t, s)


def _cond(t):
    """K = |e0||e1| / |N| per triangle ((n, 3, 3) vertices)."""
    e0, e1 = t[:, 1] - t[:, 0], t[:, 2] - t[:, 0]
    return np.linalg.norm(e0, axis=1) * np.linalg.norm(e1, axis=1) / np.linalg.norm(np.cross(e0, e1), axis=1)


def _proven_eta(A, B, d):
    """The per-pair bound DESIGN.md 4.2 proves for the filter's excess over the
    true distance: 5.2e-8 sqrt(L (|w| + L)) + 6.7e-16 K |w| + rounding, with
    |w| <= d + 2L (L = max edge, K = max conditioning of the two faces)."""
    edge = np.maximum(np.linalg.norm(A - np.roll(A, -1, 1), axis=2).max(1),
                      np.linalg.norm(B - np.roll(B, -1, 1), axis=2).max(1))
    scale = np.maximum(np.abs(A).max((1, 2)), np.abs(B).max((1, 2)))

    w = d + 2 * edge
    return 5.2e-8 * np.sqrt(edge * (w + edge)) + 6.7e-16 * np.maximum(_cond(A), _cond(B)) * w + 1e-13 * scale, edge, scale


@pytest.mark.parametrize("seed", [11, 12])
def test_filter_error_within_eta_at_scale(seed):
    """The filter's value against the reference composition on 10M adversarial
    pairs per seed: never above d + eta_proven (what the exact pass's band
    relies on), never below d by more than the 2^-20 high-word truncation."""
    worst_hi = 0.0
    overshoot = 0
    for part in range(5):
        a, b = adversarial_pairs(seed * 100 + part, 2_000_000)
        ref = T.pairs_distance(a, b)
        if part == 0 and O.REF is not None:  # the device composition is the reference's, slivers included
            idx = np.random.default_rng(seed).choice(len(a), 200_000, replace=False)
            r0 = O.ref_pairs_distance(a[idx], b[idx])
            r0 = r0[:, 0] if r0.ndim > 1 else r0
            assert np.array_equal(np.float64(ref[idx]).view(np.uint64), np.float64(r0).view(np.uint64))
        d2 = T.pairs_filter(a, b)
        fin = np.isfinite(ref)
        assert np.array_equal(np.isfinite(d2), fin)  # same degenerate skips
        assert fin.mean() > 0.9
        dt, r = np.sqrt(d2[fin]), ref[fin]
        A, B = a[fin].reshape(-1, 3, 3), b[fin].reshape(-1, 3, 3)
        eta, edge, scale = _proven_eta(A, B, r)
        hi = (dt - r) / eta                                  # excess over the proven bound
        k = int(np.argmax(hi))
        assert hi[k] <= 1.0, (hi[k], A[k].ravel(), B[k].ravel(), r[k], dt[k])
        # below the reference: d~ is a distance between two real points (or 0
        # for a certified crossing), so it can only undershoot the TRUE distance
        # by the high-word truncation. The reference composition itself
        # overshoots the true distance on some pairs: slivers (Eberly's
        # det = a00 a11 - a01^2 cancels, kernels.cpp:144-217) and crossings
        # whose edge is parallel to the other plane below its 1e-12 threshold
        # (kernels.cpp:243-244). That side is harmless for the band (it only
        # flags more pairs). Every pair below d_ref beyond the truncation is
        # checked against the exact rational distance (tests/exact_tt.py).
        # truncation: |h| to its high word, then d~^2 to its high word (2 x 2^-21
        # relative on d~), plus a vertex projection misread on a face of
        # conditioning K (6.7e-16 K |w|)
        trunc = 2e-6 * r + 1e-12 * scale + (eta - 5.2e-8 * np.sqrt(edge * (r + 3 * edge)))
        lo = (r - dt) / trunc
        for j in np.argsort(-lo)[:12]:
            if lo[j] <= 1.0:
                break
            true = float(ET.tri_tri_distance2(A[j].ravel(), B[j].ravel())) ** 0.5
            assert true - dt[j] <= 2e-6 * true + trunc[j] - 2e-6 * r[j], (A[j].ravel(), B[j].ravel(), dt[j], r[j], true)
            overshoot += r[j] > true
        worst_hi = max(worst_hi, hi[k])
    print(f"seed {seed}: 10M pairs, max (d~ - d)/eta_proven = {worst_hi:.3g}; "
          f"{overshoot} pairs where the reference overshoots the exact distance (d~ matches the exact one)")


@pytest.mark.parametrize("seed", [13, 14])
def test_filter_f32_error_within_eta_at_scale(seed):
    """FULL mode's candidate set with the FP32 edge/edge candidates
    (tdb_pairs_filter_f32: edge32_kernel's arithmetic relative to b's box
    centre) on 10M adversarial pairs per seed: d~ never above d + eta_proven +
    eta_f32_proven. Each pair is centred on its b triangle and
    the pairs are grouped by edge-length decade, so the origin radius rB of a
    call is that of its own pairs (production: B's box). The library also
    evaluates the packed form (edge_pair32x2, two A edges per f32x2 op) and
    returns NaN for a pair whose packed values differ from the scalar ones in
    any bit, so the isfinite assertion pins the packed kernel to this bound."""
    u = 2.0 ** -24
    worst = 0.0
    for part in range(5):
        a, b = adversarial_pairs(seed * 100 + part, 2_000_000)
        c = np.tile(b.reshape(-1, 3, 3).mean(1), 3)
        a, b = np.ascontiguousarray(a - c), np.ascontiguousarray(b - c)
        ref = T.pairs_distance(a, b)
        fin = np.isfinite(ref)
        A3, B3 = a.reshape(-1, 3, 3), b.reshape(-1, 3, 3)
        edge = np.maximum(np.linalg.norm(A3 - np.roll(A3, -1, 1), axis=2).max(1),
                          np.linalg.norm(B3 - np.roll(B3, -1, 1), axis=2).max(1))
        dec = np.floor(np.log10(np.maximum(edge, 1e-300)))
        for dv in np.unique(dec[fin]):
            idx = np.nonzero(fin & (dec == dv))[0]
            d2, _, rB = T.pairs_filter_f32(a[idx], b[idx])
            assert np.isfinite(d2).all()
            dt, r = np.sqrt(d2), ref[idx]
            eta, e, _ = _proven_eta(A3[idx], B3[idx], r)
            X = 12 * u * e * (r + 3 * e)              # the FP32 solve's squared excess, |w| <= d + 2L
            solve = np.where(r > 0.5 * np.sqrt(X), X / (2 * np.maximum(r, 1e-300)), np.sqrt(X))
            lin = u * (2 * rB + 10 * (r + 4 * e))     # float data, w and the evaluation
            hi = (dt - r) / (eta + solve + lin)
            k = int(np.argmax(hi))
            assert hi[k] <= 1.0, (hi[k], dv, a[idx][k], b[idx][k], r[k], dt[k])
            worst = max(worst, float(hi[k]))
    print(f"seed {seed}: 10M pairs, max (d~ - d)/(eta_proven + eta_f32_proven) = {worst:.3g}")


@pytest.mark.parametrize("seed", [21, 22])
def test_intersects_cull_margin_at_scale(seed):
    """hit_kernel (plane cull + exact survivors) == the exact predicate on
    every pair: 400k one-face records around one literal face."""
    rng = np.random.default_rng(seed)
    lit = np.array([[0, 0, 0, 1, 0, 0, 0, 1, 0]], float)
    n = 400_000
    k = n // 4
    # grazing: b crosses or just misses a's plane / edges by 10^-15..10^-3
    g = 10.0 ** rng.uniform(-15, -3, (k, 1)) * rng.choice([-1, 1], (k, 1))
    p = rng.uniform(-0.2, 1.2, (k, 3))
    p[:, 2] = 0
    b1 = np.concatenate([p + [0, 0, 1], p + g * [0, 0, 1] + rng.normal(scale=0.3, size=(k, 3)) * [1, 1, 0],
                         p + [0.1, 0.2, 0] + g * [0, 0, 1]], 1)
    # edge-on: b's edge runs through a's edges at tiny offsets
    q = rng.uniform(-0.2, 1.2, (k, 3)) * [1, 1, 0]
    e = 10.0 ** rng.uniform(-15, -3, (k, 1)) * rng.normal(size=(k, 3))
    b2 = np.concatenate([q + e, q + [0, 0, 1] + e, q + rng.normal(size=(k, 3))], 1)
    # near-coplanar overlaps
    b3 = rng.uniform(-0.5, 1.5, (k, 9))
    b3[:, 2::3] = 10.0 ** rng.uniform(-15, -6, (k, 1)) * rng.normal(size=(k, 3))
    # vertex touches: one vertex of b on a (interior / edge) +- tiny
    u, v = rng.random(n - 3 * k), rng.random(n - 3 * k)
    v = v * (1 - u)
    c = np.stack([u, v, 10.0 ** rng.uniform(-15, -3, len(u)) * rng.choice([-1, 1], len(u))], 1)
    b4 = np.concatenate([c, c + rng.normal(size=c.shape) + [0, 0, 1], c + rng.normal(size=c.shape) + [0, 0, 1]], 1)
    recs = np.concatenate([b1, b2, b3, b4])
    # shared random rigid motion / scale / offset for literal and every record (the cull's tau
    # scales with the object AABB and |coord|)
    R = _rots(rng, 1)[0]
    s = 10.0 ** rng.integers(-2, 3)
    t = rng.uniform(-1, 1, 3) * (1e6 if seed % 2 else 3.0)
    place = lambda m: ((m.reshape(-1, 3) @ R.T) * s + t).reshape(-1, 9)
    lit_p, recs_p = place(lit), place(recs)
    off = np.arange(n + 1, dtype=np.uint64)
    hit, hp = T.table_eval(T.OP_INTERSECTS, T.Table(recs_p, off), T.Mesh(lit_p))
    exact = T.pairs_intersects(recs_p, np.repeat(lit_p, n, 0))
    print(f"seed {seed}: {n} pairs, {exact.sum()} hits")
    assert 0 < exact.sum() < n
    assert np.array_equal(hit, exact), np.flatnonzero(hit != exact)[:10]
    assert (hp[hit] == 0).all() and (hp[~hit] == np.iinfo(np.uint64).max).all()


@pytest.mark.parametrize("seed", [31, 32])
def test_segment_queries_near_edges_bit_exact(seed):
    """distance_to_mesh for segments passing within 1e-14..1e-3 of a mesh
    edge (shared by two faces: exact ties and near ties), through the fused
    query kernel's candidate lists and band, against the pinned oracle."""
    import os

    import oracle as O
    from conftest import bits

    rng = np.random.default_rng(seed)
    m = T.unit_sphere(2000)                                # 2,048 faces, shared edges
    m = (m.reshape(-1, 3) * 10.0 ** rng.uniform(-2, 2) + rng.uniform(-1, 1, 3) * 1e4).reshape(-1, 9)
    n = 100_000
    tri = m[rng.integers(0, len(m), n)].reshape(-1, 3, 3)
    j = rng.integers(0, 3, n)
    e0 = tri[np.arange(n), j]
    e1 = tri[np.arange(n), (j + 1) % 3]
    L = np.linalg.norm(e1 - e0, axis=1, keepdims=True)
    p = e0 + rng.uniform(-0.1, 1.1, (n, 1)) * (e1 - e0)
    ed = (e1 - e0) / L
    dirn = rng.normal(size=(n, 3))
    dirn -= (dirn * ed).sum(1, keepdims=True) * ed * rng.uniform(0.0, 1.0, (n, 1))  # from crossing to near-parallel
    dirn /= np.linalg.norm(dirn, axis=1, keepdims=True)
    off = np.cross(ed, dirn)
    off /= np.linalg.norm(off, axis=1, keepdims=True) + 1e-300
    c = p + off * (10.0 ** rng.uniform(-14, -3, (n, 1))) * L * rng.choice([-1, 1], (n, 1))
    h = rng.uniform(0.05, 1.0, (n, 1)) * L
    segs = np.concatenate([c - h * dirn, c + h * dirn], 1)
    dd, ff = T.segments_mesh_distance(segs, m)
    rd, rf = O.segments_mesh_distance(segs, m, threads=os.cpu_count())
    bad = np.flatnonzero((bits(dd) != bits(rd)) | (ff != rf))
    assert len(bad) == 0, (len(bad), bad[:5], dd[bad[:5]], rd[bad[:5]], ff[bad[:5]], rf[bad[:5]])
    hh, hf = T.segments_mesh_intersects(segs, m)
    rh, rhf = O.segments_mesh_intersects(segs, m, threads=os.cpu_count())
    assert np.array_equal(hh.astype(bool), rh.astype(bool)) and np.array_equal(hf, rhf)


_BATCH_SCRIPT = r"""
import sys
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + '/tests')
import numpy as np
import oracle as O
import paper_1808_09571_b200 as T
from conftest import bits, GOLDEN
T.init(0)
z = np.load(GOLDEN + '/meshes.npz'); cases = {}
for k in z.files:
    name, f = k.split('/'); cases.setdefault(name, {})[f] = z[k]
for name, c in cases.items():
    r = T.mesh_mesh_distance(c['a'], c['b'])
    assert bits(r.distance) == bits(c['dist']), name
    assert (r.pair_index if r.pair_index is not None else O.U64_MAX) == int(c['pair']), name
    if r.pair_index is not None:
        assert np.array_equal(bits(np.array(r.closest_on_b)), bits(c['on_b'])), name
    h = T.mesh_mesh_intersects(c['a'], c['b'])
    assert h.hit == bool(c['hit']) and (h.pair_index if h.hit else O.U64_MAX) == int(c['hit_pair']), name
t = dict(np.load(GOLDEN + '/table.npz'))
tab, q = T.Table(t['table'], t['offsets']), T.Mesh(t['query'])
d, dp = T.table_eval(T.OP_DISTANCE, tab, q)
assert np.array_equal(bits(d), bits(t['dist'])) and np.array_equal(dp, t['dist_pair'])
hh, hp = T.table_eval(T.OP_INTERSECTS, tab, q)
assert np.array_equal(hh, t['hit'].astype(bool)) and np.array_equal(hp, t['hit_pair'])
s = T.unit_sphere(10_000)
r = T.mesh_mesh_distance(np.concatenate([T.translate(s, 0, 0, 9.0), s]), T.translate(s, 2.5, 0, 0))
assert r.distance == 0.5 and r.pair_index == O.mesh_mesh_distance(np.concatenate([T.translate(s, 0, 0, 9.0), s]), T.translate(s, 2.5, 0, 0))[1]
assert T.last_stats()['kernels'] > 20  # really split into batches
print('BATCHES OK')
"""


def test_item_cap_splits_into_batches_bit_exact():
    """With the per-launch item cap forced down (TDB_MAX_ITEMS), every call
    runs as several tile batches; merged answers must equal the golden ones."""
    import os
    import subprocess
    import sys

    from conftest import ROOT

    env = dict(os.environ, TDB_MAX_ITEMS="7")
    out = subprocess.run([sys.executable, "-c", _BATCH_SCRIPT, ROOT], env=env, capture_output=True, text=True,
                         timeout=600)
    assert "BATCHES OK" in out.stdout, out.stdout + out.stderr


@pytest.mark.parametrize("seed", [41, 42])
def test_intersects_on_reference_noise_families(seed):
    """The device culls + exact predicate == the reference itself (oracle/_ref)
    on the families where the reference's own rounding decides (slivers up to
    K = 1e13, edges 1e-12..1e-8 rad from the other plane crossing just
    outside it; tests/adversarial.py): the table path
    (hit_kernel, one object per record), the mesh x mesh lowest hit pair, and
    segment queries against a sliver soup."""
    import adversarial as AD
    import oracle as O

    if O.REF is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(seed)
    n = 60_000
    fams = [AD.sliver_literal(rng, n, w) for w in (1e-8, 1e-9, 1e-10, 1e-11, 1e-12)]
    fams += [AD.sliver_records(rng, n), AD.grazing_parallel(rng, n), AD.grazing_parallel(rng, n)]
    for k, (recs, lit) in enumerate(fams):
        ref = O.ref_pairs_intersects(recs, np.repeat(lit, n, 0)).astype(bool)
        hit, hp = T.table_eval(T.OP_INTERSECTS, T.Table(recs, np.arange(n + 1, dtype=np.uint64)), T.Mesh(lit))
        bad = np.flatnonzero(hit != ref)
        assert len(bad) == 0, (k, len(bad), recs[bad[:2]], lit)
        h = T.mesh_mesh_intersects(recs, lit)
        rh, rp = O.ref_mesh_mesh_intersects(recs, lit)
        assert h.hit == rh and (not rh or h.pair_index == rp), (k, h, rp)
        print(f"family {k}: {ref.sum()} reference hits of {n}")
    mesh, segs = AD.sliver_mesh_and_segments(rng, 2000, 100_000)
    hh, hf = T.segments_mesh_intersects(segs, mesh)
    rh, rf = O.ref_segments_mesh_intersects(segs, mesh)
    assert rh.sum() > 100
    assert np.array_equal(hh.astype(bool), rh.astype(bool)) and np.array_equal(hf, rf)
