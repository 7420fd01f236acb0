"""TEST INFRASTRUCTURE ONLY: ctypes access to the CPU checkers.

* ``C``   — ``oracle/liboracle.so``: the plain-C restatement of the
  reference primitives and of the SURVEY.md 8(a) A17 triangle-pair
  composition (tindb_oracle.c).
* ``REF`` — ``oracle/_ref/libtindb_ref.so``: the unmodified reference
  sources (/root/reference/proj/src/kernels.cpp, dataset.cpp, ...) plus the
  A17 composition harness (ref_composition.cpp). ``None`` when it was never
  built.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module. The product package
(``paper_1808_09571_b200``) never does.
"""
from __future__ import annotations

import ctypes as ct
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_C = os.path.join(HERE, "liboracle.so")
LIB_REF = os.path.join(HERE, "_ref", "libtindb_ref.so")

_D = ct.POINTER(ct.c_double)
_U64 = ct.POINTER(ct.c_uint64)
_U8 = ct.POINTER(ct.c_uint8)


class OrDist(ct.Structure):
    _fields_ = [("d", ct.c_double), ("on_a", ct.c_double * 3), ("on_b", ct.c_double * 3)]


class OrMeshDist(ct.Structure):
    _fields_ = [
        ("d", ct.c_double),
        ("pair", ct.c_uint64),
        ("found", ct.c_int),
        ("on_a", ct.c_double * 3),
        ("on_b", ct.c_double * 3),
    ]


def _dp(a):
    return a.ctypes.data_as(_D)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _load_c():
    if not os.path.exists(LIB_C):
        return None
    L = ct.CDLL(LIB_C)
    L.or_tri_tri_distance.argtypes = [_D, _D, ct.POINTER(OrDist)]
    L.or_tri_tri_intersects.argtypes = [_D, _D]
    L.or_pairs_distance.argtypes = [_D, _D, ct.c_uint64, _D]
    L.or_pairs_intersects.argtypes = [_D, _D, ct.c_uint64, _U8]
    L.or_segment_segment_distance.argtypes = [_D, _D, ct.POINTER(OrDist)]
    L.or_point_triangle_distance.argtypes = [_D, _D, ct.POINTER(OrDist)]
    L.or_segment_triangle_distance.argtypes = [_D, _D, ct.POINTER(OrDist)]
    L.or_segment_triangle_intersect.argtypes = [_D, _D]
    L.or_triangle_is_degenerate.argtypes = [_D]
    L.or_mesh_mesh_distance.argtypes = [_D, ct.c_uint64, _D, ct.c_uint64, ct.c_uint64,
                                        ct.c_uint64, ct.c_uint64, ct.c_int,
                                        ct.POINTER(OrMeshDist)]
    L.or_mesh_mesh_intersects.argtypes = [_D, ct.c_uint64, _D, ct.c_uint64, ct.c_uint64,
                                          ct.c_uint64, ct.c_uint64, ct.c_int, _U64]
    L.or_mesh_mesh_distance_pruned.argtypes = [_D, ct.c_uint64, _D, ct.c_uint64, ct.c_double, ct.c_int,
                                               ct.POINTER(OrMeshDist)]
    L.or_mesh_mesh_intersects_pruned.argtypes = [_D, ct.c_uint64, _D, ct.c_uint64, ct.c_int, _U64]
    for fn in ("or_segments_mesh_distance", "or_points_mesh_distance"):
        getattr(L, fn).argtypes = [_D, ct.c_uint64, _D, ct.c_uint64, ct.c_int, _D, _U64]
    L.or_segments_mesh_intersects.argtypes = [_D, ct.c_uint64, _D, ct.c_uint64, ct.c_int, _U8, _U64]
    L.or_table_distance.argtypes = [_D, _U64, ct.c_uint64, _D, ct.c_uint64, ct.c_int, _D, _U64]
    L.or_table_intersects.argtypes = [_D, _U64, ct.c_uint64, _D, ct.c_uint64, ct.c_int, _U8,
                                      _U64]
    return L


def _load_ref():
    if not os.path.exists(LIB_REF):
        return None
    L = ct.CDLL(LIB_REF)
    L.ref_segment_segment_distance.argtypes = [_D, _D, _D]
    L.ref_point_triangle_distance.argtypes = [_D, _D, _D]
    L.ref_segment_triangle_distance.argtypes = [_D, _D, _D]
    L.ref_segment_triangle_intersect.argtypes = [_D, _D]
    L.ref_triangle_is_degenerate.argtypes = [_D]
    L.ref_pairs_distance.argtypes = [_D, _D, ct.c_uint64, _D]
    L.ref_pairs_intersects.argtypes = [_D, _D, ct.c_uint64, _U8]
    L.ref_mesh_mesh_distance.argtypes = [_D, ct.c_uint64, _D, ct.c_uint64, ct.c_uint64,
                                         ct.c_uint64, ct.c_uint64, ct.c_int, _D, _U64]
    L.ref_mesh_mesh_intersects.argtypes = [_D, ct.c_uint64, _D, ct.c_uint64, ct.c_uint64,
                                           ct.c_uint64, ct.c_uint64, ct.c_int, _U64]
    L.ref_unit_sphere.argtypes = [ct.c_uint64, _D]
    L.ref_unit_sphere.restype = ct.c_uint64
    L.ref_ore_body.argtypes = [ct.c_uint64, _D]
    L.ref_ore_body.restype = ct.c_uint64
    L.ref_queries_mesh_distance_flag.argtypes = [ct.c_int, _D, ct.c_uint64, _D, ct.c_uint64, ct.c_int, ct.c_int, _D,
                                                 _U64]
    L.ref_terrain.argtypes = [ct.c_uint32, ct.c_uint32, ct.c_double, ct.c_uint64, _D]
    L.ref_terrain.restype = ct.c_uint64
    L.ref_random_triangles.argtypes = [ct.c_uint64, ct.c_uint64, ct.c_double, ct.c_double, _D]
    for fn in ("ref_segments_mesh_distance", "ref_points_mesh_distance"):
        getattr(L, fn).argtypes = [_D, ct.c_uint64, _D, ct.c_uint64, ct.c_int, _D, _U64]
    L.ref_segments_mesh_intersects.argtypes = [_D, ct.c_uint64, _D, ct.c_uint64, ct.c_int, _U8, _U64]
    L.ref_make_drills.argtypes = [ct.c_uint64, ct.c_uint64, ct.c_int, _D]
    L.ref_make_drills.restype = ct.c_uint64
    L.ref_mesh_volume.argtypes = [_D, ct.c_uint64, ct.c_uint64, ct.POINTER(ct.c_int)]
    L.ref_mesh_volume.restype = ct.c_double
    L.ref_unit_cube.argtypes = [_D]
    L.ref_unit_cube.restype = ct.c_uint64
    L.ref_parse_wkt.argtypes = [ct.c_char_p, ct.c_uint64, ct.POINTER(ct.c_int), _D, ct.c_uint64, _U64,
                                ct.POINTER(ct.c_int), ct.c_char_p, ct.c_uint64, _U64]
    L.ref_parse_wkt.restype = ct.c_int
    L.ref_serialize_mesh.argtypes = [_D, ct.c_uint64, ct.c_char_p, ct.c_uint64]
    L.ref_serialize_mesh.restype = ct.c_uint64
    return L


C = _load_c()
REF = _load_ref()

U64_MAX = (1 << 64) - 1


# ---------------------------------------------------------------- C oracle
def pairs_distance(a, b):
    """A17 distance for aligned pair arrays a[k], b[k] (k x 9)."""
    a, b = _f64(a).reshape(-1, 9), _f64(b).reshape(-1, 9)
    out = np.empty(len(a), np.float64)
    C.or_pairs_distance(_dp(a), _dp(b), len(a), _dp(out))
    return out


def pairs_intersects(a, b):
    a, b = _f64(a).reshape(-1, 9), _f64(b).reshape(-1, 9)
    out = np.empty(len(a), np.uint8)
    C.or_pairs_intersects(_dp(a), _dp(b), len(a), out.ctypes.data_as(_U8))
    return out.astype(bool)


def tri_tri_distance(a9, b9):
    a9, b9 = _f64(a9), _f64(b9)
    o = OrDist()
    C.or_tri_tri_distance(_dp(a9), _dp(b9), ct.byref(o))
    return o.d, np.array(o.on_a[:]), np.array(o.on_b[:])


def mesh_mesh_distance(a, b, threads=None, rows=None):
    """(dist, pair, found, on_a, on_b). rows = (begin, end, stride) or None."""
    a, b = _f64(a).reshape(-1, 9), _f64(b).reshape(-1, 9)
    r0, r1, rs = rows if rows else (0, len(a), 1)
    o = OrMeshDist()
    C.or_mesh_mesh_distance(_dp(a), len(a), _dp(b), len(b), r0, r1, rs,
                            threads or os.cpu_count() or 1, ct.byref(o))
    return o.d, o.pair, bool(o.found), np.array(o.on_a[:]), np.array(o.on_b[:])


def mesh_mesh_intersects(a, b, threads=None, rows=None):
    """(hit, lowest hit pair or U64_MAX)."""
    a, b = _f64(a).reshape(-1, 9), _f64(b).reshape(-1, 9)
    r0, r1, rs = rows if rows else (0, len(a), 1)
    p = ct.c_uint64(0)
    C.or_mesh_mesh_intersects(_dp(a), len(a), _dp(b), len(b), r0, r1, rs,
                              threads or os.cpu_count() or 1, ct.byref(p))
    return p.value != U64_MAX, p.value


def mesh_mesh_distance_pruned(a, b, ub, threads=None):
    """Exact (dist, pair, found, on_a, on_b) among pairs with distance <= ub
    (the full answer whenever ub >= the true minimum), AABB-pruned."""
    a, b = _f64(a).reshape(-1, 9), _f64(b).reshape(-1, 9)
    o = OrMeshDist()
    C.or_mesh_mesh_distance_pruned(_dp(a), len(a), _dp(b), len(b), float(ub),
                                   threads or os.cpu_count() or 1, ct.byref(o))
    return o.d, o.pair, bool(o.found), np.array(o.on_a[:]), np.array(o.on_b[:])


def mesh_mesh_intersects_pruned(a, b, threads=None):
    """Exact (hit, lowest hit pair), AABB-pruned."""
    a, b = _f64(a).reshape(-1, 9), _f64(b).reshape(-1, 9)
    p = ct.c_uint64(0)
    C.or_mesh_mesh_intersects_pruned(_dp(a), len(a), _dp(b), len(b), threads or os.cpu_count() or 1,
                                     ct.byref(p))
    return p.value != U64_MAX, p.value


def _queries(lib, prefix, kind, q, mesh, threads):
    width = 3 if kind == "points" else 6
    q = _f64(q).reshape(-1, width)
    mesh = _f64(mesh).reshape(-1, 9)
    face = np.empty(len(q), np.uint64)
    th = threads or os.cpu_count() or 1
    if kind == "intersects":
        hit = np.empty(len(q), np.uint8)
        getattr(lib, prefix + "segments_mesh_intersects")(_dp(q), len(q), _dp(mesh), len(mesh), th,
                                                          hit.ctypes.data_as(_U8), face.ctypes.data_as(_U64))
        return hit.astype(bool), face
    d = np.empty(len(q), np.float64)
    getattr(lib, prefix + f"{kind}_mesh_distance")(_dp(q), len(q), _dp(mesh), len(mesh), th, _dp(d),
                                                   face.ctypes.data_as(_U64))
    return d, face


def segments_mesh_distance(segs, mesh, threads=None):
    """(distance, face) per segment: distance_to_mesh (kernels.cpp:388)."""
    return _queries(C, "or_", "segments", segs, mesh, threads)


def points_mesh_distance(pts, mesh, threads=None):
    return _queries(C, "or_", "points", pts, mesh, threads)


def segments_mesh_intersects(segs, mesh, threads=None):
    """(hit, face) per segment: intersects_mesh (kernels.cpp:407)."""
    return _queries(C, "or_", "intersects", segs, mesh, threads)


def ref_segments_mesh_distance(segs, mesh, threads=None):
    return _queries(REF, "ref_", "segments", segs, mesh, threads)


def ref_points_mesh_distance(pts, mesh, threads=None):
    return _queries(REF, "ref_", "points", pts, mesh, threads)


def ref_segments_mesh_intersects(segs, mesh, threads=None):
    return _queries(REF, "ref_", "intersects", segs, mesh, threads)


def ref_queries_mesh_distance_flag(q, mesh, has_degenerate_faces, points=False, threads=None):
    """distance_to_mesh per query with the mesh's has_degenerate_faces set to
    the given value (not refreshed): kernels.cpp:350,357."""
    q = _f64(q).reshape(-1, 3 if points else 6)
    m = _f64(mesh).reshape(-1, 9)
    d, f = np.empty(len(q)), np.empty(len(q), np.uint64)
    REF.ref_queries_mesh_distance_flag(1 if points else 0, _dp(q), len(q), _dp(m), len(m),
                                       threads or os.cpu_count() or 1, 1 if has_degenerate_faces else 0,
                                       _dp(d), f.ctypes.data_as(_U64))
    return d, f


def ref_make_drills(seed, count, style=0):
    out = np.empty((count, 6), np.float64)
    REF.ref_make_drills(seed, count, style, _dp(out))
    return out


def table_eval(op, table, offsets, query, threads=None):
    """Per record: (dist or hit array, pair array). op in {'distance','intersects'}."""
    table, query = _f64(table).reshape(-1, 9), _f64(query).reshape(-1, 9)
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    nobj = len(offsets) - 1
    pair = np.empty(nobj, np.uint64)
    th = threads or os.cpu_count() or 1
    if op == "distance":
        d = np.empty(nobj, np.float64)
        C.or_table_distance(_dp(table), offsets.ctypes.data_as(_U64), nobj, _dp(query),
                            len(query), th, _dp(d), pair.ctypes.data_as(_U64))
        return d, pair
    h = np.empty(nobj, np.uint8)
    C.or_table_intersects(_dp(table), offsets.ctypes.data_as(_U64), nobj, _dp(query),
                          len(query), th, h.ctypes.data_as(_U8), pair.ctypes.data_as(_U64))
    return h.astype(bool), pair


# ------------------------------------------------------- reference (_ref)
def ref_pairs_distance(a, b):
    a, b = _f64(a).reshape(-1, 9), _f64(b).reshape(-1, 9)
    out = np.empty((len(a), 7), np.float64)
    REF.ref_pairs_distance(_dp(a), _dp(b), len(a), _dp(out))
    return out


def ref_pairs_intersects(a, b):
    a, b = _f64(a).reshape(-1, 9), _f64(b).reshape(-1, 9)
    out = np.empty(len(a), np.uint8)
    REF.ref_pairs_intersects(_dp(a), _dp(b), len(a), out.ctypes.data_as(_U8))
    return out.astype(bool)


def ref_mesh_mesh_distance(a, b, threads=None, rows=None):
    a, b = _f64(a).reshape(-1, 9), _f64(b).reshape(-1, 9)
    r0, r1, rs = rows if rows else (0, len(a), 1)
    out = np.empty(7, np.float64)
    p = ct.c_uint64(0)
    REF.ref_mesh_mesh_distance(_dp(a), len(a), _dp(b), len(b), r0, r1, rs,
                               threads or os.cpu_count() or 1, _dp(out), ct.byref(p))
    return out[0], p.value, p.value != U64_MAX, out[1:4].copy(), out[4:7].copy()


def ref_mesh_mesh_intersects(a, b, threads=None, rows=None):
    a, b = _f64(a).reshape(-1, 9), _f64(b).reshape(-1, 9)
    r0, r1, rs = rows if rows else (0, len(a), 1)
    p = ct.c_uint64(0)
    REF.ref_mesh_mesh_intersects(_dp(a), len(a), _dp(b), len(b), r0, r1, rs,
                                 threads or os.cpu_count() or 1, ct.byref(p))
    return p.value != U64_MAX, p.value


def ref_unit_sphere(face_target):
    n = REF.ref_unit_sphere(face_target, None)
    out = np.empty((n, 9), np.float64)
    REF.ref_unit_sphere(face_target, _dp(out))
    return out


def ref_ore_body(face_target):
    n = REF.ref_ore_body(face_target, None)
    out = np.empty((n, 9), np.float64)
    REF.ref_ore_body(face_target, _dp(out))
    return out


def ref_terrain(nx=1024, ny=512, amp=20.0, seed=42):
    """C2's terrain over the reference's Rng (ref_composition.cpp ref_terrain)."""
    n = REF.ref_terrain(nx, ny, ct.c_double(amp), seed, None)
    out = np.empty((n, 9), np.float64)
    REF.ref_terrain(nx, ny, ct.c_double(amp), seed, _dp(out))
    return out


def ref_random_triangles(seed, n, lo=-1.0, hi=1.0):
    out = np.empty((n, 9), np.float64)
    REF.ref_random_triangles(seed, n, lo, hi, _dp(out))
    return out


def ref_mesh_volume(tris, chunk=4096):
    """(volume, closed) from the reference mesh_volume (kernels.cpp:27-46)."""
    t = _f64(tris).reshape(-1, 9)
    c = ct.c_int(0)
    v = REF.ref_mesh_volume(_dp(t), len(t), chunk, ct.byref(c))
    return v, bool(c.value)


def ref_unit_cube():
    out = np.empty((12, 9), np.float64)
    REF.ref_unit_cube(_dp(out))
    return out


class RefWktError(ValueError):
    """tindb::WktParseError raised by the reference parser (wkt.hpp:13)."""

    def __init__(self, what, position):
        super().__init__(what)
        self.what = what
        self.position = position


REF_KINDS = {0: "point", 1: "segment", 2: "linestring", 3: "mesh"}


def ref_parse_wkt(text):
    """The reference parse_wkt (wkt.cpp:188): (kind, coords, mesh_source) or
    raises RefWktError(what, position). Mesh coords are (n, 9)."""
    raw = text.encode() if isinstance(text, str) else bytes(text)
    kind, src, n = ct.c_int(0), ct.c_int(0), ct.c_uint64(0)
    pos = ct.c_uint64(0)
    err = ct.create_string_buffer(512)
    cap = 9 * (raw.count(b",") + 4)  # >= 9 doubles per point listed
    out = np.empty(cap, np.float64)
    rc = REF.ref_parse_wkt(raw, len(raw), ct.byref(kind), _dp(out), cap, ct.byref(n), ct.byref(src), err, 512,
                           ct.byref(pos))
    if rc:
        raise RefWktError(err.value.decode(), pos.value)
    k = REF_KINDS[kind.value]
    if k == "mesh":
        return k, out[: 9 * n.value].reshape(-1, 9).copy(), ("tin", "polyhedralsurface")[src.value]
    return k, out[: 3 * n.value].reshape(-1, 3).copy(), None


def ref_serialize_mesh(tris, as_bytes=False):
    """The reference serialize_wkt(TriangleMesh) text (canonical TIN Z)."""
    t = _f64(tris).reshape(-1, 9)
    n = REF.ref_serialize_mesh(_dp(t), len(t), None, 0)
    buf = ct.create_string_buffer(n)
    REF.ref_serialize_mesh(_dp(t), len(t), buf, n)
    raw = buf.raw[:n]
    return raw if as_bytes else raw.decode()


def sha_f64(a):
    """sha256 of a float64 array's bytes (golden fixture digests)."""
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a, np.float64).tobytes()).hexdigest()
