"""tindb_b200 — Python mirror of the triangle-pair operator API.

A thin ctypes layer over ``libtindb_b200.so`` (the C ABI in
``include/tindb_b200.h``). Names follow the reference operator surface
(``tindb::kernels``, /root/reference/proj/include/tindb/kernels.hpp and
batch.hpp): ``mesh_mesh_distance`` / ``mesh_mesh_intersects`` are the new
Mesh x Mesh entries beside ``distance_to_mesh`` / ``intersects_mesh``, and
``run_batch`` mirrors ``kernels::run_batch`` (batch.hpp:49) for a mesh table
against a mesh literal.

There is no CPU fallback: importing works without a GPU (so the ABI can be
checked), but every compute call raises ``RuntimeError`` unless an sm_100
device is present and the library was built (``python __graft_entry__.py``
or ``make``).
"""
from __future__ import annotations

import ctypes as ct
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence, Union

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtindb_b200.so")

TDB_OK, TDB_E_ARG, TDB_E_CUDA, TDB_E_NOMEM, TDB_E_PARSE = 0, -1, -2, -3, -4
OP_DISTANCE, OP_INTERSECTS = 1, 2
MODE_FULL, MODE_CULL = 0, 1
U64_MAX = (1 << 64) - 1

_D = ct.POINTER(ct.c_double)
_U64 = ct.POINTER(ct.c_uint64)
_U8 = ct.POINTER(ct.c_uint8)


class DistOut(ct.Structure):
    _fields_ = [
        ("distance", ct.c_double),
        ("pair", ct.c_uint64),
        ("i", ct.c_uint64),
        ("j", ct.c_uint64),
        ("on_a", ct.c_double * 3),
        ("on_b", ct.c_double * 3),
        ("found", ct.c_int32),
        ("_pad", ct.c_int32),
    ]


class HitOut(ct.Structure):
    _fields_ = [
        ("hit", ct.c_int32),
        ("_pad", ct.c_int32),
        ("pair", ct.c_uint64),
        ("i", ct.c_uint64),
        ("j", ct.c_uint64),
    ]


class FaceResult(ct.Structure):
    """tdb_face_result: the reference's per-face DistanceResult /
    IntersectionResult (kernels.hpp:28-48) for one query and one triangle."""
    _fields_ = [
        ("distance", ct.c_double),
        ("on_query", ct.c_double * 3),
        ("on_face", ct.c_double * 3),
        ("t", ct.c_double),
        ("u", ct.c_double),
        ("v", ct.c_double),
        ("w", ct.c_double),
        ("hit", ct.c_int32),
        ("_pad", ct.c_int32),
        ("point", ct.c_double * 3),
    ]


class Stats(ct.Structure):
    _fields_ = [
        ("ms_total", ct.c_double),
        ("ms_filter", ct.c_double),
        ("ms_verify", ct.c_double),
        ("pairs", ct.c_uint64),
        ("items", ct.c_uint64),
        ("items_flagged", ct.c_uint64),
        ("candidates", ct.c_uint64),
        ("exact_pairs", ct.c_uint64),
        ("kernels", ct.c_uint64),
        ("pairs_evaluated", ct.c_uint64),
        ("near_degenerate", ct.c_uint64),
        ("rounds", ct.c_int32),
        ("_pad", ct.c_int32),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if not k.startswith("_")}


# (name, restype, argtypes) for every entry point of include/tindb_b200.h
_SIGS = [
    ("tdb_init", ct.c_int, [ct.c_int]),
    ("tdb_set_stream", ct.c_int, [ct.c_void_p]),
    ("tdb_set_mode", ct.c_int, [ct.c_int]),
    ("tdb_last_error", ct.c_char_p, []),
    ("tdb_last_stats", ct.c_int, [ct.POINTER(Stats)]),
    ("tdb_last_near_degenerate", ct.c_int, [_U64, ct.c_uint64, _U64]),
    ("tdb_device_count", ct.c_int, []),
    ("tdb_mesh_upload", ct.c_int, [_D, ct.c_uint64, ct.POINTER(ct.c_void_p)]),
    ("tdb_table_upload", ct.c_int, [_D, _U64, ct.c_uint64, ct.POINTER(ct.c_void_p)]),
    ("tdb_geom_info", ct.c_int, [ct.c_void_p, _U64, _U64, _U64, _D]),
    ("tdb_geom_feature_counts", ct.c_int, [ct.c_void_p, _U64, _U64, _U64, _U64, _U64, _U64]),
    ("tdb_mesh_from_wkt", ct.c_int, [ct.c_char_p, ct.c_uint64, ct.POINTER(ct.c_void_p), _U64]),
    ("tdb_table_from_wkt", ct.c_int, [ct.c_char_p, _U64, ct.c_uint64, ct.POINTER(ct.c_void_p), _U64, _U64]),
    ("tdb_geom_download", ct.c_int, [ct.c_void_p, _D]),
    ("tdb_geom_offsets", ct.c_int, [ct.c_void_p, _U64]),
    ("tdb_geom_set_has_degenerate_faces", ct.c_int, [ct.c_void_p, _U8, ct.c_uint64]),
    ("tdb_mesh_free", None, [ct.c_void_p]),
    ("tdb_table_free", None, [ct.c_void_p]),
    ("tdb_mesh_mesh_distance", ct.c_int, [ct.c_void_p, ct.c_void_p, ct.POINTER(DistOut)]),
    ("tdb_mesh_mesh_intersects", ct.c_int, [ct.c_void_p, ct.c_void_p, ct.POINTER(HitOut)]),
    ("tdb_mesh_mesh_distance_rows", ct.c_int,
     [ct.c_void_p, ct.c_uint64, ct.c_uint64, ct.c_void_p, ct.POINTER(DistOut)]),
    ("tdb_mesh_mesh_intersects_rows", ct.c_int,
     [ct.c_void_p, ct.c_uint64, ct.c_uint64, ct.c_void_p, ct.POINTER(HitOut)]),
    ("tdb_table_eval", ct.c_int, [ct.c_int, ct.c_void_p, ct.c_void_p, _D, _U8, _U64]),
    ("tdb_table_eval_rows", ct.c_int,
     [ct.c_int, ct.c_void_p, ct.c_uint64, ct.c_uint64, ct.c_void_p, _D, _U8, _U64]),
    ("tdb_distance_host", ct.c_int, [_D, ct.c_uint64, _D, ct.c_uint64, ct.POINTER(DistOut)]),
    ("tdb_intersects_host", ct.c_int, [_D, ct.c_uint64, _D, ct.c_uint64, ct.POINTER(HitOut)]),
    ("tdb_pairs_distance", ct.c_int, [_D, _D, ct.c_uint64, _D]),
    ("tdb_pairs_intersects", ct.c_int, [_D, _D, ct.c_uint64, _U8]),
    ("tdb_pairs_filter", ct.c_int, [_D, _D, ct.c_uint64, _D]),
    ("tdb_pairs_filter_f32", ct.c_int, [_D, _D, ct.c_uint64, _D, _D]),
    ("tdb_gen_unit_sphere", ct.c_uint64, [ct.c_uint64, _D]),
    ("tdb_gen_ore_body", ct.c_uint64, [ct.c_uint64, _D]),
    ("tdb_gen_terrain", ct.c_uint64, [ct.c_uint32, ct.c_uint32, ct.c_double, ct.c_uint64, _D]),
    ("tdb_fp64_peak", ct.c_int, [_D, _D]),
    ("tdb_mesh_volume", ct.c_int, [ct.c_void_p, ct.c_uint64, _D]),
    ("tdb_table_volume", ct.c_int, [ct.c_void_p, ct.c_uint64, _D]),
    ("tdb_literal_table_eval", ct.c_int, [ct.c_int, ct.c_int, _D, ct.c_void_p, _D, _U8, _U64]),
    ("tdb_segments_mesh_distance", ct.c_int, [_D, ct.c_uint64, ct.c_void_p, _D, _U64]),
    ("tdb_points_mesh_distance", ct.c_int, [_D, ct.c_uint64, ct.c_void_p, _D, _U64]),
    ("tdb_segments_mesh_intersects", ct.c_int, [_D, ct.c_uint64, ct.c_void_p, _U8, _U64]),
    ("tdb_gen_drills", ct.c_uint64, [ct.c_uint64, ct.c_uint64, ct.c_int, _D]),
    ("tdb_queries_upload", ct.c_int, [_D, ct.c_uint64, ct.c_int, ct.POINTER(ct.c_void_p)]),
    ("tdb_queries_free", None, [ct.c_void_p]),
    ("tdb_queries_mesh_distance", ct.c_int, [ct.c_void_p, ct.c_void_p, _D, _U64]),
    ("tdb_queries_mesh_intersects", ct.c_int, [ct.c_void_p, ct.c_void_p, _U8, _U64]),
    ("tdb_query_face_result", ct.c_int, [ct.c_int, ct.c_int, _D, _D, ct.POINTER(FaceResult)]),
    ("tdb_group_create", ct.c_int, [ct.c_int, ct.POINTER(ct.c_int), ct.POINTER(ct.c_void_p)]),
    ("tdb_group_free", None, [ct.c_void_p]),
    ("tdb_group_size", ct.c_int, [ct.c_void_p]),
    ("tdb_group_mesh_upload", ct.c_int, [ct.c_void_p, _D, ct.c_uint64, ct.POINTER(ct.c_void_p)]),
    ("tdb_group_table_upload", ct.c_int, [ct.c_void_p, _D, _U64, ct.c_uint64, ct.POINTER(ct.c_void_p)]),
    ("tdb_gmesh_free", None, [ct.c_void_p]),
    ("tdb_group_mesh_mesh_distance", ct.c_int, [ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.POINTER(DistOut)]),
    ("tdb_group_mesh_mesh_intersects", ct.c_int, [ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.POINTER(HitOut)]),
    ("tdb_group_table_eval", ct.c_int, [ct.c_void_p, ct.c_int, ct.c_void_p, ct.c_void_p, _D, _U8, _U64]),
    ("tdb_group_last_stats", ct.c_int, [ct.c_void_p, ct.c_int, ct.POINTER(Stats)]),
]
EXPORTS = [s[0] for s in _SIGS]

_lib = None


def lib():
    """The loaded C ABI library (raises if it was never built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built: run `python __graft_entry__.py` (or make)")
        L = ct.CDLL(LIB_PATH)
        for name, res, args in _SIGS:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class TdbError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"tindb_b200 error {code}: {msg}")
        self.code = code


def _check(rc):
    if rc != TDB_OK:
        msg = lib().tdb_last_error()
        msg = msg.decode() if msg else ""
        if rc == TDB_E_ARG:
            raise ValueError(msg)  # kernels.cpp:403 std::invalid_argument
        raise TdbError(rc, msg)


def _f64(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.size % 9:
        raise ValueError("triangle arrays hold 9 doubles per face")
    return a.reshape(-1, 9)


def _dp(a):
    return a.ctypes.data_as(_D)


def init(device: int = 0):
    _check(lib().tdb_init(device))


def device_count() -> int:
    return lib().tdb_device_count()


def set_stream(stream_handle: Optional[int]):
    """Launch on a caller stream (e.g. torch.cuda.current_stream().cuda_stream)."""
    _check(lib().tdb_set_stream(ct.c_void_p(stream_handle or 0)))


def set_mode(mode: int):
    _check(lib().tdb_set_mode(mode))


def last_stats() -> dict:
    s = Stats()
    _check(lib().tdb_last_stats(ct.byref(s)))
    return s.as_dict()


NEAR_LOG_CAP = 1024  # kNearLogCap (exact.cuh): entries kept per call


def last_near_degenerate(cap: int = NEAR_LOG_CAP):
    """(count, entries[k, 2]) of the near-degenerate pairs the exact pass met
    in the last call on this thread: (object, pair) per entry (object = A
    object / table row / query; pair = i*|B|+j / face index). `count` may
    exceed the entries kept (1024)."""
    buf = np.zeros((max(cap, 0), 2), np.uint64)
    cnt = np.zeros(1, np.uint64)
    _check(lib().tdb_last_near_degenerate(buf.ctypes.data_as(_U64), cap, cnt.ctypes.data_as(_U64)))
    n = int(cnt[0])
    return n, buf[: min(n, cap, NEAR_LOG_CAP)]


class _Geom:
    """Device-resident triangle store (SoA planes + per-object AABB headers)."""

    def __init__(self, handle):
        self._h = ct.c_void_p(handle)

    @property
    def handle(self):
        return self._h

    def info(self):
        n, no, nd = ct.c_uint64(), ct.c_uint64(), ct.c_uint64()
        box = (ct.c_double * 6)()
        _check(lib().tdb_geom_info(self._h, ct.byref(n), ct.byref(no), ct.byref(nd), box))
        return {"faces": n.value, "objects": no.value, "degenerate": nd.value, "aabb": list(box)}

    def feature_counts(self):
        """The distance filter's shared candidates: as the B
        side, total non-degenerate faces, distinct vertices and distinct edges
        over the store's 64-face blocks; as the A side, the distinct edges and
        vertices of its super-tiles (tile_edges, tile_vertices); the distinct
        edges per 8,192 faces (super_edges, B's lists in large calls)."""
        f, v, e, te, tv, se = (ct.c_uint64() for _ in range(6))
        _check(lib().tdb_geom_feature_counts(self._h, ct.byref(f), ct.byref(v), ct.byref(e), ct.byref(te),
                                             ct.byref(tv), ct.byref(se)))
        return {"faces": f.value, "vertices": v.value, "edges": e.value, "tile_edges": te.value,
                "tile_vertices": tv.value, "super_edges": se.value}

    def download(self) -> np.ndarray:
        """The stored faces as (n, 9) float64, face order (the AoS the store was built from)."""
        n = self.info()["faces"]
        out = np.empty((n, 9), np.float64)
        _check(lib().tdb_geom_download(self._h, _dp(out)))
        return out

    def set_has_degenerate_faces(self, flags) -> "_Geom":
        """TriangleMesh::has_degenerate_faces per object (geometry.hpp:84):
        point / segment distance queries skip an object's degenerate faces
        only when its flag is set (kernels.cpp:350,357). A bool applies to
        every object."""
        n = self.info()["objects"]
        f = np.broadcast_to(np.asarray(flags, dtype=np.uint8), (n,)).copy()
        _check(lib().tdb_geom_set_has_degenerate_faces(self._h, f.ctypes.data_as(_U8), n))
        return self

    def free(self):
        if self._h is not None and self._h.value:
            lib().tdb_mesh_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Mesh(_Geom):
    """A TriangleMesh uploaded to HBM (geometry.hpp:81-98 layout, 72 B/face)."""

    def __init__(self, triangles):
        t = _f64(triangles)
        h = ct.c_void_p()
        _check(lib().tdb_mesh_upload(_dp(t), len(t), ct.byref(h)))
        super().__init__(h.value)
        self.faces = len(t)


class Table(_Geom):
    """A mesh column (GeometryRecord rows, store_types.hpp:14-32) in HBM."""

    def __init__(self, triangles, face_offsets, ids: Optional[Sequence[int]] = None):
        t = _f64(triangles)
        off = np.ascontiguousarray(face_offsets, dtype=np.uint64)
        h = ct.c_void_p()
        _check(lib().tdb_table_upload(_dp(t), off.ctypes.data_as(_U64), len(off) - 1, ct.byref(h)))
        super().__init__(h.value)
        self.objects = len(off) - 1
        self.ids = list(ids) if ids is not None else list(range(1, self.objects + 1))


class WktParseError(ValueError):
    """tindb::WktParseError (wkt.hpp:13-23): the reference's what() and 0-based
    byte `position` within the literal; `literal` indexes the rejected literal
    of a multi-literal load."""

    def __init__(self, what: str, position: int, literal: int = 0):
        super().__init__(what)
        self.what = what
        self.position = position
        self.literal = literal


def _wkt_bytes(text) -> bytes:
    return text.encode() if isinstance(text, str) else bytes(text)


def mesh_from_wkt(text) -> Mesh:
    """parse_wkt (wkt.hpp:35) of a TIN Z / POLYHEDRALSURFACE Z literal, parsed
    on the device straight into the store (bit-identical coordinates)."""
    raw = _wkt_bytes(text)
    h, pos = ct.c_void_p(), ct.c_uint64(0)
    rc = lib().tdb_mesh_from_wkt(raw, len(raw), ct.byref(h), ct.byref(pos))
    if rc == TDB_E_PARSE:
        raise WktParseError(lib().tdb_last_error().decode(), pos.value, 0)
    _check(rc)
    m = Mesh.__new__(Mesh)
    _Geom.__init__(m, h.value)
    m.faces = m.info()["faces"]
    return m


def table_from_wkt(literals: Sequence, ids: Optional[Sequence[int]] = None) -> Table:
    """A mesh column from WKT literals (load_csv_text's WKT field,
    store.cpp:71-122), all parsed in one device pass; object i = literal i."""
    raws = [_wkt_bytes(x) for x in literals]
    off = np.zeros(len(raws) + 1, np.uint64)
    off[1:] = np.cumsum([len(r) for r in raws], dtype=np.uint64)
    blob = b"".join(raws)
    h, lit, pos = ct.c_void_p(), ct.c_uint64(0), ct.c_uint64(0)
    rc = lib().tdb_table_from_wkt(blob, off.ctypes.data_as(_U64), len(raws), ct.byref(h), ct.byref(lit),
                                  ct.byref(pos))
    if rc == TDB_E_PARSE:
        raise WktParseError(lib().tdb_last_error().decode(), pos.value, lit.value)
    _check(rc)
    t = Table.__new__(Table)
    _Geom.__init__(t, h.value)
    t.objects = len(raws)
    t.ids = list(ids) if ids is not None else list(range(1, t.objects + 1))
    return t


@dataclass
class DistanceResult:
    """kernels::DistanceResult (kernels.hpp:28-34) for a triangle pair winner."""
    distance: float
    pair_index: Optional[int]
    face_a: Optional[int]
    face_b: Optional[int]
    closest_on_a: tuple
    closest_on_b: tuple


@dataclass
class IntersectionResult:
    """kernels::IntersectionResult (kernels.hpp:43-48) with the lowest hit pair."""
    hit: bool
    pair_index: Optional[int]
    face_a: Optional[int]
    face_b: Optional[int]


def _dist_result(o: DistOut) -> DistanceResult:
    f = bool(o.found)
    return DistanceResult(o.distance, o.pair if f else None, o.i if f else None, o.j if f else None,
                          tuple(o.on_a), tuple(o.on_b))


def _hit_result(o: HitOut) -> IntersectionResult:
    h = bool(o.hit)
    return IntersectionResult(h, o.pair if h else None, o.i if h else None, o.j if h else None)


def _as_mesh(x) -> Mesh:
    return x if isinstance(x, _Geom) else Mesh(x)


def mesh_mesh_distance(a, b, rows: Optional[tuple] = None) -> DistanceResult:
    """ST_3DDistance(a, b) over every triangle pair."""
    a, b = _as_mesh(a), _as_mesh(b)
    o = DistOut()
    if rows is None:
        _check(lib().tdb_mesh_mesh_distance(a.handle, b.handle, ct.byref(o)))
    else:
        _check(lib().tdb_mesh_mesh_distance_rows(a.handle, rows[0], rows[1], b.handle, ct.byref(o)))
    return _dist_result(o)


def mesh_mesh_intersects(a, b, rows: Optional[tuple] = None) -> IntersectionResult:
    """ST_3DIntersects(a, b): lowest intersecting pair (kernels.cpp:407-432)."""
    a, b = _as_mesh(a), _as_mesh(b)
    o = HitOut()
    if rows is None:
        _check(lib().tdb_mesh_mesh_intersects(a.handle, b.handle, ct.byref(o)))
    else:
        _check(lib().tdb_mesh_mesh_intersects_rows(a.handle, rows[0], rows[1], b.handle, ct.byref(o)))
    return _hit_result(o)


def distance_host(a, b) -> DistanceResult:
    """One-shot: host arrays in, result out (upload + evaluate + free)."""
    a, b = _f64(a), _f64(b)
    o = DistOut()
    _check(lib().tdb_distance_host(_dp(a), len(a), _dp(b), len(b), ct.byref(o)))
    return _dist_result(o)


def intersects_host(a, b) -> IntersectionResult:
    a, b = _f64(a), _f64(b)
    o = HitOut()
    _check(lib().tdb_intersects_host(_dp(a), len(a), _dp(b), len(b), ct.byref(o)))
    return _hit_result(o)


def table_eval(op: int, table: Table, literal, objects: Optional[tuple] = None):
    """Per record: (values, pair indices); values are distances or booleans."""
    lit = _as_mesh(literal)
    o0, o1 = objects if objects is not None else (0, table.objects)
    k = o1 - o0
    pair = np.empty(k, np.uint64)
    if op == OP_DISTANCE:
        d = np.empty(k, np.float64)
        _check(lib().tdb_table_eval_rows(op, table.handle, o0, o1, lit.handle, _dp(d), None,
                                         pair.ctypes.data_as(_U64)))
        return d, pair
    h = np.empty(k, np.uint8)
    _check(lib().tdb_table_eval_rows(op, table.handle, o0, o1, lit.handle, None,
                                     h.ctypes.data_as(_U8), pair.ctypes.data_as(_U64)))
    return h.astype(bool), pair


@dataclass
class KernelResult:
    """kernels::KernelResult (batch.hpp:27-32): record id + value."""
    record_id: int
    value: Union[float, bool]


def run_batch(op: int, records: Table, argument) -> List[KernelResult]:
    """kernels::run_batch (batch.hpp:49-51) for a Mesh column x Mesh literal:
    one result per record, in record order."""
    vals, _ = table_eval(op, records, argument)
    conv = float if op == OP_DISTANCE else bool
    return [KernelResult(rid, conv(v)) for rid, v in zip(records.ids, vals)]


def pairs_distance(a, b) -> np.ndarray:
    """Exact A17 composition for aligned pairs (a[k], b[k]) on the device."""
    a, b = _f64(a), _f64(b)
    out = np.empty(len(a), np.float64)
    _check(lib().tdb_pairs_distance(_dp(a), _dp(b), len(a), _dp(out)))
    return out


def pairs_intersects(a, b) -> np.ndarray:
    a, b = _f64(a), _f64(b)
    out = np.empty(len(a), np.uint8)
    _check(lib().tdb_pairs_intersects(_dp(a), _dp(b), len(a), out.ctypes.data_as(_U8)))
    return out.astype(bool)


def pairs_filter(a, b) -> np.ndarray:
    """The roofline kernel's FP64 filter value d~^2 for aligned pairs."""
    a, b = _f64(a), _f64(b)
    out = np.empty(len(a), np.float64)
    _check(lib().tdb_pairs_filter(_dp(a), _dp(b), len(a), _dp(out)))
    return out


def pairs_filter_f32(a, b):
    """FULL mode's candidate set for aligned pairs (FP64 vertex/face, FP32
    edge/edge relative to b's box centre): (d~^2 per pair, origin, rB).
    A pair whose packed FP32 candidates (edge_pair32x2) differ from the scalar
    ones in any bit gets NaN."""
    a, b = _f64(a), _f64(b)
    out = np.empty(len(a), np.float64)
    orb = np.empty(4, np.float64)
    _check(lib().tdb_pairs_filter_f32(_dp(a), _dp(b), len(a), _dp(out), _dp(orb)))
    return out, orb[:3].copy(), float(orb[3])


def _qarr(q, width):
    q = np.ascontiguousarray(q, dtype=np.float64)
    if q.size % width:
        raise ValueError(f"queries hold {width} doubles each")
    return q.reshape(-1, width)


QUERY_SEGMENTS, QUERY_POINTS = 0, 1


class Queries:
    """A device-resident column of segments (6 doubles) or points (3)."""

    def __init__(self, q, kind=QUERY_SEGMENTS):
        a = _qarr(q, 6 if kind == QUERY_SEGMENTS else 3)
        h = ct.c_void_p()
        _check(lib().tdb_queries_upload(_dp(a), len(a), kind, ct.byref(h)))
        self._h, self.n, self.kind = h, len(a), kind

    @property
    def handle(self):
        return self._h

    def free(self):
        if self._h is not None and self._h.value:
            lib().tdb_queries_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def queries_mesh_distance(q: Queries, mesh):
    """distance_to_mesh per resident query: (distance, face) arrays."""
    m = _as_mesh(mesh)
    d, f = np.empty(q.n), np.empty(q.n, np.uint64)
    _check(lib().tdb_queries_mesh_distance(q.handle, m.handle, _dp(d), f.ctypes.data_as(_U64)))
    return d, f


def queries_mesh_intersects(q: Queries, mesh):
    """intersects_mesh per resident segment: (hit, lowest hit face) arrays."""
    m = _as_mesh(mesh)
    h, f = np.empty(q.n, np.uint8), np.empty(q.n, np.uint64)
    _check(lib().tdb_queries_mesh_intersects(q.handle, m.handle, h.ctypes.data_as(_U8), f.ctypes.data_as(_U64)))
    return h.view(bool), f  # 0/1 bytes: a zero-copy bool view


def segments_mesh_distance(segments, mesh):
    """distance_to_mesh(segment, mesh) per segment (kernels.cpp:388):
    (distance array, face index array; UINT64_MAX = none)."""
    if isinstance(segments, Queries):
        return queries_mesh_distance(segments, mesh)
    s, m = _qarr(segments, 6), _as_mesh(mesh)
    d, f = np.empty(len(s)), np.empty(len(s), np.uint64)
    _check(lib().tdb_segments_mesh_distance(_dp(s), len(s), m.handle, _dp(d), f.ctypes.data_as(_U64)))
    return d, f


def points_mesh_distance(points, mesh):
    """distance_to_mesh(point, mesh) per point (kernels.cpp:382)."""
    if isinstance(points, Queries):
        return queries_mesh_distance(points, mesh)
    p, m = _qarr(points, 3), _as_mesh(mesh)
    d, f = np.empty(len(p)), np.empty(len(p), np.uint64)
    _check(lib().tdb_points_mesh_distance(_dp(p), len(p), m.handle, _dp(d), f.ctypes.data_as(_U64)))
    return d, f


def segments_mesh_intersects(segments, mesh):
    """intersects_mesh(segment, mesh) per segment (kernels.cpp:407):
    (hit array, lowest hit face array)."""
    if isinstance(segments, Queries):
        return queries_mesh_intersects(segments, mesh)
    s, m = _qarr(segments, 6), _as_mesh(mesh)
    h, f = np.empty(len(s), np.uint8), np.empty(len(s), np.uint64)
    _check(lib().tdb_segments_mesh_intersects(_dp(s), len(s), m.handle, h.ctypes.data_as(_U8),
                                              f.ctypes.data_as(_U64)))
    return h.astype(bool), f


def query_face_result(op: int, query, tri) -> FaceResult:
    """The reference's full per-face result (closest points + params, or hit
    point + params) for one segment (6 doubles) or point (3) and one
    triangle (9), evaluated on the device."""
    q = np.ascontiguousarray(query, dtype=np.float64).ravel()
    t = np.ascontiguousarray(tri, dtype=np.float64).ravel()
    if t.size != 9 or q.size not in (3, 6):
        raise ValueError("query is 3 or 6 doubles, the triangle 9")
    o = FaceResult()
    _check(lib().tdb_query_face_result(op, QUERY_POINTS if q.size == 3 else QUERY_SEGMENTS, _dp(q), _dp(t),
                                       ct.byref(o)))
    return o


def drills(count: int, seed: int = 42, style: int = 0) -> np.ndarray:
    """make_drills (dataset.cpp:141-165): style 0 vertical jittered, 1 uniform."""
    out = np.empty((count, 6), np.float64)
    lib().tdb_gen_drills(seed, count, style, _dp(out))
    return out


def mesh_volume(mesh, chunk_size: int = 4096) -> float:
    """ST_3DVolume: kernels::mesh_volume (kernels.cpp:27-46) bit for bit, for
    the same ExecutorConfig::chunk_size (permissive policy)."""
    m = _as_mesh(mesh)
    v = ct.c_double()
    _check(lib().tdb_mesh_volume(m.handle, chunk_size, ct.byref(v)))
    return v.value


def table_volume(table: Table, chunk_size: int = 4096) -> np.ndarray:
    """run_batch(Volume) over a mesh column: mesh_volume per object, each with
    its own chunk tree (batch.cpp:23-29), bit for bit."""
    out = np.empty(table.objects, np.float64)
    _check(lib().tdb_table_volume(table.handle, chunk_size, _dp(out)))
    return out


# ---- mesh generators (host; bit-identical to dataset.cpp) -------------------
def unit_sphere(face_target: int) -> np.ndarray:
    n = lib().tdb_gen_unit_sphere(face_target, None)
    out = np.empty((n, 9), np.float64)
    lib().tdb_gen_unit_sphere(face_target, _dp(out))
    return out


def ore_body(face_target: int) -> np.ndarray:
    n = lib().tdb_gen_ore_body(face_target, None)
    out = np.empty((n, 9), np.float64)
    lib().tdb_gen_ore_body(face_target, _dp(out))
    return out


def terrain(nx: int = 1024, ny: int = 512, amp: float = 20.0, seed: int = 42) -> np.ndarray:
    n = lib().tdb_gen_terrain(nx, ny, amp, seed, None)
    out = np.empty((n, 9), np.float64)
    lib().tdb_gen_terrain(nx, ny, amp, seed, _dp(out))
    return out


def translate(tris, dx=0.0, dy=0.0, dz=0.0) -> np.ndarray:
    """Per-vertex translation (fixtures.cpp:37-46 translated)."""
    t = _f64(tris).copy()
    t[:, 0::3] += dx
    t[:, 1::3] += dy
    t[:, 2::3] += dz
    return t


def fp64_peak() -> tuple:
    """(TFLOP/s, ms) of the DFMA issue-rate microbenchmark on this device."""
    tf, ms = ct.c_double(), ct.c_double()
    _check(lib().tdb_fp64_peak(ct.byref(tf), ct.byref(ms)))
    return tf.value, ms.value


def literal_table_eval(op: int, literal, table: Table):
    """run_batch with a segment (6 doubles) or point (3) literal over a mesh
    column: per record distance_to_mesh / intersects_mesh (batch.cpp:44-48,
    :59). Returns (dist or hit, face) per record; face = U64_MAX when none."""
    lit = np.ascontiguousarray(literal, dtype=np.float64).reshape(-1)
    kind = {6: QUERY_SEGMENTS, 3: QUERY_POINTS}.get(lit.size)
    if kind is None:
        raise ValueError("a literal is a segment (6 doubles) or a point (3)")
    face = np.empty(table.objects, np.uint64)
    if op == OP_DISTANCE:
        d = np.empty(table.objects, np.float64)
        _check(lib().tdb_literal_table_eval(op, kind, _dp(lit), table.handle, _dp(d), None, face.ctypes.data_as(_U64)))
        return d, face
    h = np.empty(table.objects, np.uint8)
    _check(lib().tdb_literal_table_eval(op, kind, _dp(lit), table.handle, None, h.ctypes.data_as(_U8),
                                        face.ctypes.data_as(_U64)))
    return h.astype(bool), face


# --------------------------------------------------------------------------
# device group: one process, several GPUs (include/tindb_b200.h tdb_group_*)
# --------------------------------------------------------------------------
class _GroupGeom:
    def __init__(self, group, handle, faces, objects):
        self.group, self._h, self.faces, self.objects = group, ct.c_void_p(handle), faces, objects

    @property
    def handle(self):
        return self._h

    def free(self):
        if self._h is not None and self._h.value:
            lib().tdb_gmesh_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Group:
    """Several devices driven from this process: replicated geometry, A rows
    (or table objects) split over the members, one NCCL MIN all-reduce."""

    def __init__(self, devices: Union[int, Sequence[int]]):
        devs = list(range(devices)) if isinstance(devices, int) else list(devices)
        arr = (ct.c_int * len(devs))(*devs)
        h = ct.c_void_p()
        _check(lib().tdb_group_create(len(devs), arr, ct.byref(h)))
        self._h, self.devices = h, devs

    @property
    def handle(self):
        return self._h

    def __len__(self):
        return lib().tdb_group_size(self._h)

    def mesh(self, triangles) -> _GroupGeom:
        t = _f64(triangles)
        h = ct.c_void_p()
        _check(lib().tdb_group_mesh_upload(self._h, _dp(t), len(t), ct.byref(h)))
        return _GroupGeom(self, h.value, len(t), 1)

    def table(self, triangles, face_offsets) -> _GroupGeom:
        t = _f64(triangles)
        off = np.ascontiguousarray(face_offsets, dtype=np.uint64)
        h = ct.c_void_p()
        _check(lib().tdb_group_table_upload(self._h, _dp(t), off.ctypes.data_as(_U64), len(off) - 1, ct.byref(h)))
        return _GroupGeom(self, h.value, len(t), len(off) - 1)

    def mesh_mesh_distance(self, a: _GroupGeom, b: _GroupGeom) -> DistanceResult:
        o = DistOut()
        _check(lib().tdb_group_mesh_mesh_distance(self._h, a.handle, b.handle, ct.byref(o)))
        return _dist_result(o)

    def mesh_mesh_intersects(self, a: _GroupGeom, b: _GroupGeom) -> IntersectionResult:
        o = HitOut()
        _check(lib().tdb_group_mesh_mesh_intersects(self._h, a.handle, b.handle, ct.byref(o)))
        return _hit_result(o)

    def table_eval(self, op: int, records: _GroupGeom, literal: _GroupGeom):
        k = records.objects
        pair = np.empty(k, np.uint64)
        if op == OP_DISTANCE:
            d = np.empty(k, np.float64)
            _check(lib().tdb_group_table_eval(self._h, op, records.handle, literal.handle, _dp(d), None,
                                              pair.ctypes.data_as(_U64)))
            return d, pair
        h = np.empty(k, np.uint8)
        _check(lib().tdb_group_table_eval(self._h, op, records.handle, literal.handle, None,
                                          h.ctypes.data_as(_U8), pair.ctypes.data_as(_U64)))
        return h.astype(bool), pair

    def last_stats(self, member: int) -> dict:
        st = Stats()
        _check(lib().tdb_group_last_stats(self._h, member, ct.byref(st)))
        return st.as_dict()

    def free(self):
        if self._h is not None and self._h.value:
            lib().tdb_group_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
