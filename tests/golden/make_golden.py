"""Regenerate tests/golden/*.npz from the REFERENCE itself.

Runs the unmodified reference sources compiled by oracle/Makefile
(oracle/_ref/libtindb_ref.so: kernels.cpp, dataset.cpp, fixtures.cpp + the
A17 composition harness ref_composition.cpp). Needs /root/reference, so it
only runs in the build container; the .npz outputs are committed and travel
to the GPU box.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def rot(rng):
    q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    return q


def xf(tri9, R, t):
    v = tri9.reshape(3, 3) @ R.T + t
    return v.reshape(9)


def adversarial(seed=7):
    """Hand-built degenerate-adjacent triangle pairs, each in several rigid
    placements (random rotation + offset, including offsets of 1e6)."""
    rng = np.random.default_rng(seed)
    base = np.array([0, 0, 0, 1, 0, 0, 0, 1, 0], float)
    cases = []

    def add(a, b):
        cases.append((np.asarray(a, float), np.asarray(b, float)))

    add(base, base)                                            # identical (coplanar)
    add(base, base + np.array([0.3, 0.2, 0] * 3))              # coplanar overlap
    add(base, base + np.array([2.0, 0, 0] * 3))                # coplanar apart
    add(base, [0, 0, 0, -1, 0, 0.5, 0, -1, 0.3])               # shared vertex
    add(base, [0, 0, 0, 1, 0, 0, 0.3, 0.2, 1.0])               # shared edge (hinge)
    add(base, [0.2, 0.2, 0, 0.5, 0.5, 1, 0.1, 0.6, 1])         # vertex touches interior
    add(base, [0.2, 0.2, -1, 0.3, 0.2, 1, 0.25, 0.9, 0.5])     # proper crossing
    add(base, [0.5, -0.5, 1e-9, 0.5, 0.5, 1e-9, 3, 3, 5])      # edge grazes just above
    add(base, [0, 0, 1, 1, 0, 1, 0, 1, 1])                     # parallel stacked
    add(base, [0, 0, 1, 1, 1e-14, 1, 0, 1, 1])                 # near-parallel stacked
    add(base, [0.5, 0.5, 0, 1.5, 0.5, 0, 1.5, -0.5, 1])        # vertex on hypotenuse
    add(base, [0.25, 0.25, 1e-13, 0.75, 0.25, -1e-13, 0.5, 0.75, 1e-13])  # near-coplanar crossing
    add(base, [2, 0, 0, 3, 0, 0, 2, 1, 0])                     # collinear-edge apart
    add(base, [1, 0, 0, 2, 0, 0, 1.5, 0, 1])                   # touching vertex, perpendicular
    add(base, [0.5, 0, -1, 0.5, 0, 1, 0.6, 0, 0.5])            # b in plane y=0 crossing edge
    add(base, [1, 1, 0, 2, 2, 0, 1, 2, 0])                     # coplanar vertex contact at distance
    tiny = 1.2e-15
    add(base, [5, 5, 5, 5 + tiny, 5, 5, 5, 5 + tiny, 5])       # near the 1e-30 area^2 threshold
    add(base, [5, 5, 5, 5 + 1e-16, 5, 5, 5, 5 + 1e-16, 5])     # degenerate by threshold
    add(base, [5, 5, 5, 6, 6, 6, 7, 7, 7])                     # exactly collinear (degenerate)
    add(base, [0.1, 0.1, 0.0, 0.9, 0.1, 0.0, 0.1, 0.9, 0.0])   # b inside a (coplanar)
    add([0, 0, 0, 1, 0, 0, 0, 0, 1], [0, 0, 0, 0, 1, 0, 0, 0, 1])  # hinge on z axis
    a_list, b_list = [], []
    for a, b in cases:
        a_list.append(a)
        b_list.append(b)
        for k in range(6):
            R = rot(rng)
            t = rng.uniform(-3, 3, 3) if k < 3 else rng.uniform(-1, 1, 3) * 1e6
            s = 10.0 ** rng.integers(-3, 4)
            a_list.append(xf(a * s, R, t))
            b_list.append(xf(b * s, R, t))
    # near-parallel edge pairs at graded angles
    for ang in [0.0, 1e-16, 1e-13, 1e-10, 1e-8, 1e-6, 1e-4, 1e-2]:
        for sep in [0.0, 1e-12, 1e-6, 0.1]:
            a = np.array([0, 0, 0, 1, 0, 0, 0.5, -1, -0.3], float)
            b = np.array([0.2, sep, 0, 1.2, sep + ang, 0, 0.7, 1, 0.4], float)
            a_list.append(a)
            b_list.append(b)
    return np.array(a_list), np.array(b_list)


def clustered(seed, n):
    """Random pairs at small separations: many near-touching/crossing pairs."""
    rng = np.random.default_rng(seed)
    a = O.ref_random_triangles(seed, n)
    b = O.ref_random_triangles(seed + 1, n) * 0.3
    c = a.reshape(n, 3, 3).mean(axis=1)
    b = b + np.tile(c + rng.normal(scale=0.05, size=(n, 3)), 3)
    return a, b


def mesh_cases():
    s80, s320, s1280 = O.ref_unit_sphere(80), O.ref_unit_sphere(320), O.ref_unit_sphere(1000)
    cube = O.ref_unit_cube()

    def tr(m, dx=0.0, dy=0.0, dz=0.0):
        t = m.copy()
        t[:, 0::3] += dx
        t[:, 1::3] += dy
        t[:, 2::3] += dz
        return t

    rng = np.random.default_rng(11)
    soup_a = O.ref_random_triangles(101, 300)
    soup_b = O.ref_random_triangles(102, 250) * 0.5 + 0.7
    deg = soup_a[:60].copy()
    deg[::7, 3:6] = deg[::7, 0:3]          # zero-length edge -> degenerate faces
    ore = O.ref_ore_body(1000)
    # the terrain generator is new (not in the reference): inputs come from
    # the product's host generator, outputs from the reference composition
    import paper_1808_09571_b200 as T
    ter = T.terrain(16, 8, 20.0, 42)
    cases = {
        "spheres_offset_2.5": (s80, tr(s80, 2.5)),
        "spheres_1280_offset_2.5": (s1280, tr(s1280, 2.5)),
        "nested_0.9": (s320, s320 * 0.9),
        "spheres_shift_0.5": (s320, tr(s320, 0.5)),
        "spheres_shift_0.37_diag": (s320, tr(s320, 0.37, 0.21, -0.1)),
        "cube_touching_face": (cube, tr(cube, 1.0)),
        "cube_gap": (cube, tr(cube, 1.25, 0.5, 0.5)),
        "cube_overlap": (cube, tr(cube, 0.5, 0.5, 0.5)),
        "cube_same": (cube, cube.copy()),
        "soups": (soup_a, soup_b),
        "soup_with_degenerate": (deg, soup_b[:80]),
        "ore_vs_sphere": (ore, tr(s320 * 50.0, 500.0, 500.0, -20.0)),
    }
    cases["terrain_vs_ore"] = (ter, ore)
    out = {}
    for name, (a, b) in cases.items():
        d, p, found, wa, wb = O.ref_mesh_mesh_distance(a, b, threads=8)
        hit, hp = O.ref_mesh_mesh_intersects(a, b, threads=8)
        out[name] = dict(a=a, b=b, dist=np.float64(d), pair=np.uint64(p), found=found,
                         on_a=wa, on_b=wb, hit=hit, hit_pair=np.uint64(hp))
    return out


def table_case():
    """20 records (spheres/cubes placed around a query sphere) x query."""
    rng = np.random.default_rng(5)
    q = O.ref_unit_sphere(320)
    objs = []
    for r in range(20):
        base = O.ref_unit_sphere(80) if r % 3 else O.ref_unit_cube()
        s = rng.uniform(0.1, 0.6)
        c = rng.uniform(-2.0, 2.0, 3)
        m = base * s
        m[:, 0::3] += c[0]
        m[:, 1::3] += c[1]
        m[:, 2::3] += c[2]
        objs.append(m)
    objs.insert(7, np.zeros((0, 9)))  # an empty record
    off = np.cumsum([0] + [len(o) for o in objs]).astype(np.uint64)
    table = np.concatenate(objs)
    dist = np.empty(len(objs))
    dpair = np.empty(len(objs), np.uint64)
    hit = np.empty(len(objs), bool)
    hpair = np.empty(len(objs), np.uint64)
    for r, o in enumerate(objs):
        if len(o) == 0:
            dist[r], dpair[r], hit[r], hpair[r] = np.inf, O.U64_MAX, False, O.U64_MAX
            continue
        d, p, found, _, _ = O.ref_mesh_mesh_distance(o, q, threads=8)
        dist[r], dpair[r] = d, p
        hit[r], hpair[r] = O.ref_mesh_mesh_intersects(o, q, threads=8)
    return dict(table=table, offsets=off, query=q, dist=dist, dist_pair=dpair, hit=hit, hit_pair=hpair)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.float64).tobytes()).hexdigest()


def _fmt_num(rng, v):
    """One coordinate in a random textual form that still means exactly v
    (or, for the 'lossy' forms, a nearby decimal the reference rounds)."""
    k = rng.integers(0, 10)
    if k == 0:
        return repr(float(v))
    if k == 1:
        return "%.17g" % v
    if k == 2:
        return "%.17E" % v
    if k == 3:
        return "%.6e" % v                        # lossy, short
    if k == 4:
        return "%.3f" % v                        # lossy, fixed
    if k == 5:
        s = "%.25f" % v                          # long fixed
        return s
    if k == 6:
        s = repr(float(v))
        return ("00" + s) if not s.startswith("-") else "-00" + s[1:]   # leading zeros
    if k == 7:
        return "%.40e" % v                       # 41 significant digits (beyond 19)
    if k == 8:
        s = "%.3f" % v
        return s.rstrip("0") if "." in s else s   # "1." style trailing point
    return "%.0f." % v if abs(v) < 1e15 else repr(float(v))


def _ws(rng, allow_empty=True):
    opts = [" ", "  ", "\t", "\n", "\r\n", " \t "] + ([""] * 3 if allow_empty else [])
    return opts[rng.integers(0, len(opts))]


def _surface_text(rng, kw, rings):
    """TIN Z / POLYHEDRALSURFACE Z text of closed rings (lists of 3-tuples),
    with random spacing and number forms (only where the grammar allows)."""
    parts = []
    for ring in rings:
        pts = []
        for p in ring:
            a, b, c = (_fmt_num(rng, x) for x in p)
            pts.append(a + _ws(rng, False) + b + _ws(rng, False) + c)
        pts.append(pts[0])  # the closure repeats the first point's text
        sep = [_ws(rng) + "," + _ws(rng) for _ in pts[1:]]
        body = pts[0] + "".join(s + q for s, q in zip(sep, pts[1:]))
        parts.append("(" + _ws(rng) + "(" + _ws(rng) + body + _ws(rng) + ")" + _ws(rng) + ")")
    body = (_ws(rng) + "," + _ws(rng)).join(parts)
    return kw + _ws(rng, False) + "Z" + _ws(rng) + "(" + _ws(rng) + body + _ws(rng) + ")" + _ws(rng)


def wkt_cases():
    """WKT literals and what the reference's parse_wkt makes of them."""
    rng = np.random.default_rng(1808)
    texts = {}
    # reference unit tests (test_geometry.cpp:110-205)
    texts["tin_two_patches"] = "TIN Z (((0 0 0, 1 0 0, 0 1 0, 0 0 0)), ((0 0 1, 1 0 1, 0 1 1, 0 0 1)))"
    texts["tin_non_triangular"] = "TIN Z (((0 0 0, 1 0 0, 1 1 0, 0 1 0, 0 0 0)))"
    texts["poly_quad_fan"] = "POLYHEDRALSURFACE Z (((0 0 0, 1 0 0, 1 1 0, 0 1 0, 0 0 0)))"
    texts["unclosed_ring"] = "TIN Z (((0 0 0, 1 0 0, 0 1 0, 5 5 5)))"
    texts["short_ring"] = "TIN Z (((0 0 0, 1 0 0, 0 0 0)))"
    texts["no_z"] = "TIN (((0 0 0, 1 0 0, 0 1 0, 0 0 0)))"
    texts["zm"] = "TIN ZM (((0 0 0 1, 1 0 0 1, 0 1 0 1, 0 0 0 1)))"
    texts["m"] = "TIN M (((0 0 0, 1 0 0, 0 1 0, 0 0 0)))"
    texts["two_d"] = "TIN Z (((0 0, 1 0, 0 1, 0 0)))"
    texts["nan"] = "TIN Z (((0 0 nan, 1 0 0, 0 1 0, 0 0 0)))"
    texts["inf"] = "TIN Z (((inf 0 0, 1 0 0, 0 1 0, 0 0 0)))"
    texts["minus_inf"] = "TIN Z (((0 -inf 0, 1 0 0, 0 1 0, 0 0 0)))"
    texts["overflow"] = "TIN Z (((0 0 1e999, 1 0 0, 0 1 0, 0 0 0)))"
    texts["underflow"] = "TIN Z (((0 0 1e-400, 1 0 0, 0 1 0, 0 0 0)))"
    texts["trailing"] = "TIN Z (((0 0 0, 1 0 0, 0 1 0, 0 0 0))) x"
    texts["unknown_tag"] = "CIRCLE Z (0 0 0)"
    texts["empty"] = ""
    texts["blank"] = "  \n\t "
    texts["point"] = "POINT Z (1 2 3)"
    texts["linestring"] = "LINESTRING Z (0 0 0, 1 1 1)"
    texts["incomplete_triple"] = "TIN Z (((0 0 0, 1, 0 1 0, 0 0 0)))"
    texts["plus_sign"] = "TIN Z (((+1 0 0, 1 0 0, 0 1 0, +1 0 0)))"
    texts["garbage_number"] = "TIN Z (((0 0 0, 1 0 0, 0 1 x, 0 0 0)))"
    texts["interior_ring"] = "POLYHEDRALSURFACE Z (((0 0 0, 4 0 0, 4 4 0, 0 0 0), (1 1 0, 2 1 0, 2 2 0, 1 1 0)))"
    texts["missing_close"] = "TIN Z (((0 0 0, 1 0 0, 0 1 0, 0 0 0))"
    texts["extra_close"] = "TIN Z (((0 0 0, 1 0 0, 0 1 0, 0 0 0))))"
    texts["empty_surface"] = "TIN Z ()"
    texts["header_only"] = "TIN Z"
    texts["empty_patch"] = "TIN Z (())"
    texts["four_coords"] = "TIN Z (((0 0 0 0, 1 0 0, 0 1 0, 0 0 0)))"
    texts["missing_comma"] = "TIN Z (((0 0 0 1 0 0, 0 1 0, 0 0 0)))"
    texts["double_comma"] = "TIN Z (((0 0 0,, 1 0 0, 0 1 0, 0 0 0)))"
    texts["patch_no_comma"] = "TIN Z (((0 0 0, 1 0 0, 0 1 0, 0 0 0)) ((0 0 1, 1 0 1, 0 1 1, 0 0 1)))"
    texts["bad_exponent"] = "TIN Z (((0 0 1e, 1 0 0, 0 1 0, 0 0 1e)))"
    texts["dot_alone"] = "TIN Z (((0 0 ., 1 0 0, 0 1 0, 0 0 0)))"
    texts["nul_byte"] = "TIN Z (((0 0 0, 1 0\x00 0, 0 1 0, 0 0 0)))"
    texts["utf8"] = "TIN Z (((0 0 0, 1 0 0, 0 1 0, 0 0 0)))\u00a0"
    # accepted oddities of the from_chars grammar
    texts["juxtaposed"] = "TIN Z (((0-1 2, 1.5.5 -.25, 0 1 0, 0-1 2)))"
    texts["no_spaces"] = "tin z(((0 0 0,1 0 0,0 1 0,0 0 0)),((0 0 1,1 0 1,0 1 1,0 0 1)))"
    texts["case_mix"] = "  PolyhedralSurface   z\n(((0 0 0,\t1 0 0,1 1 0,0 1 0,0 0 0)))\n"
    texts["exp_forms"] = "TIN Z (((1E2 1e+2 1e-2, 1. .5 -.5, 0e0 -0 00012, 1E2 1e+2 1e-2)))"
    texts["minus_zero_closure"] = "TIN Z (((0 0 0, 1 0 0, 0 1 0, -0 -0.0 0e5)))"
    # generated meshes with random spacing and number forms
    tris = O.ref_random_triangles(77, 200, -1000.0, 1000.0)
    texts["soup_tin"] = _surface_text(rng, "TIN", [t.reshape(3, 3) for t in tris])
    polys = []
    for n in rng.integers(3, 11, 60):
        ang = np.sort(rng.uniform(0, 2 * np.pi, n))
        c = rng.uniform(-50, 50, 3)
        polys.append([c + [5 * np.cos(a), 5 * np.sin(a), rng.uniform(-1, 1)] for a in ang])
    texts["soup_poly"] = _surface_text(rng, "POLYHEDRALSURFACE", polys)
    texts["sphere_canonical"] = O.ref_serialize_mesh(O.ref_unit_sphere(1000))
    # hard decimals: exact halfway points between neighbouring doubles (hundreds
    # of digits), subnormals, near DBL_MAX
    from decimal import Decimal, getcontext
    getcontext().prec = 2000
    hard = []
    for _ in range(40):
        x = float(rng.uniform(-1e3, 1e3)) * 10.0 ** int(rng.integers(-300, 300))
        y = np.nextafter(x, np.inf)
        mid = (Decimal(x) + Decimal(float(y))) / 2
        hard.append(format(mid, "f") if abs(x) > 1e-5 and abs(x) < 1e20 else format(mid, "e"))
    hard += ["4.9406564584124654e-324", "2.4703282292062328e-324", "1.7976931348623157e308",
             "2.2250738585072011e-308", "9007199254740993", "0." + "0" * 320 + "123"]
    hard_tris = []
    for i in range(0, len(hard) - 2, 3):
        a = [hard[i], hard[i + 1], hard[i + 2]]
        hard_tris.append("((%s %s %s, 1 0 0, 0 1 0, %s %s %s))" % (*a, *a))
    texts["hard_numbers"] = "TIN Z (" + ", ".join(hard_tris) + ")"
    # an error deep inside a long literal
    big = O.ref_serialize_mesh(O.ref_unit_sphere(1000))
    cut = big.rfind("((", 0, len(big) * 2 // 3)
    texts["deep_unclosed"] = big[:cut] + "((0 0 0, 1 0 0, 0 1 0, 0 0 1))" + big[cut + len("(("):].split("))", 1)[1]

    out = {}
    for name, t in texts.items():
        try:
            kind, c, src = O.ref_parse_wkt(t)
            rec = {"text": t, "ok": True, "kind": kind}
            if kind == "mesh":
                rec.update(faces=len(c), sha=sha(c), source=src)
        except O.RefWktError as e:
            rec = {"text": t, "ok": False, "what": e.what, "position": e.position}
        out[name] = rec
    return out


def main_wkt():
    cases = wkt_cases()
    with open(os.path.join(OUT, "wkt_cases.json"), "w") as f:
        json.dump(cases, f, indent=0, sort_keys=True)
    print("wkt cases:", len(cases), "accepted:", sum(c["ok"] for c in cases.values()))


def main():
    assert O.REF is not None, "build oracle/_ref first (make -C oracle)"
    # random pairs on [-1,1]^3 (fixtures.cpp:89 random_triangle)
    a = O.ref_random_triangles(1337, 3000)
    b = O.ref_random_triangles(1338, 3000)
    ca, cb = clustered(4242, 3000)
    aa, ab = adversarial()
    A = np.concatenate([a, ca, aa])
    B = np.concatenate([b, cb, ab])
    r = O.ref_pairs_distance(A, B)
    h = O.ref_pairs_intersects(A, B)
    np.savez_compressed(os.path.join(OUT, "pairs.npz"), a=A, b=B, dist=r[:, 0], on_a=r[:, 1:4],
                        on_b=r[:, 4:7], hit=h,
                        kind=np.array([0] * 3000 + [1] * 3000 + [2] * len(aa), np.int8))
    meshes = mesh_cases()
    flat = {}
    for name, c in meshes.items():
        for k, v in c.items():
            flat[f"{name}/{k}"] = np.asarray(v)
    np.savez_compressed(os.path.join(OUT, "meshes.npz"), **flat)
    np.savez_compressed(os.path.join(OUT, "table.npz"), **table_case())
    gens = {}
    for ft in [10, 100, 1000, 10000, 100000]:
        gens[f"unit_sphere/{ft}"] = sha(O.ref_unit_sphere(ft))
        gens[f"ore_body/{ft}"] = sha(O.ref_ore_body(ft))
    with open(os.path.join(OUT, "generators.json"), "w") as f:
        json.dump(gens, f, indent=1, sort_keys=True)
    # segment / point x mesh (distance_to_mesh, intersects_mesh): the paper's
    # drill workload (make_drills, dataset.cpp:141) plus uniform segments,
    # zero-length segments and points, against a 512- and a 20,480-face ore
    drills = O.ref_make_drills(42, 3000, 0)
    unif = O.ref_make_drills(43, 2000, 1)
    zero = drills[:64].copy()
    zero[:, 3:] = zero[:, :3]
    segs = np.concatenate([drills, unif, zero])
    pts = np.random.default_rng(9).uniform([0, 0, -400], [1000, 1000, 0], (3000, 3))
    q = {"segments": segs, "points": pts}
    for name, ft in (("ore512", 500), ("ore20480", 20000)):
        ore = O.ref_ore_body(ft)
        d, f = O.ref_segments_mesh_distance(segs, ore)
        h, hf = O.ref_segments_mesh_intersects(segs, ore)
        pd, pf = O.ref_points_mesh_distance(pts, ore)
        q.update({f"{name}/mesh": ore, f"{name}/seg_dist": d, f"{name}/seg_face": f, f"{name}/seg_hit": h,
                  f"{name}/seg_hit_face": hf, f"{name}/pt_dist": pd, f"{name}/pt_face": pf})
    np.savez_compressed(os.path.join(OUT, "queries.npz"), **q)
    # mesh_volume (kernels.cpp:27-46) bits for several chunk sizes
    import paper_1808_09571_b200 as T
    vol_meshes = {"sphere_1280": O.ref_unit_sphere(1000), "ore_81920": O.ref_ore_body(100_000),
                  "cube": O.ref_unit_cube(), "terrain_16x8": T.terrain(16, 8, 20.0, 42),
                  "soup_300": O.ref_random_triangles(101, 300)}
    vols = {}
    for name, m in vol_meshes.items():
        for chunk in (1, 7, 4096):
            v, closed = O.ref_mesh_volume(m, chunk)
            vols[f"{name}/{chunk}"] = {"bits": np.float64(v).view(np.uint64).item(), "value": v, "closed": closed}
    np.savez_compressed(os.path.join(OUT, "volume_meshes.npz"), **vol_meshes)
    with open(os.path.join(OUT, "volumes.json"), "w") as f:
        json.dump(vols, f, indent=1, sort_keys=True)
    print("pairs:", len(A), "hits:", int(h.sum()), "meshes:", len(meshes))


if __name__ == "__main__":
    if sys.argv[1:] == ["wkt"]:
        main_wkt()
    else:
        main()
        main_wkt()
