// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// Thin extern "C" harness over the *unmodified* reference sources
// (/root/reference/proj/src/{kernels,dataset,wkt,closure}.cpp and
// tests/support/fixtures.cpp), compiled by oracle/Makefile with
// -Dtindb=tindb_ref into oracle/_ref/libtindb_ref.so.
//
// The reference has no mesh x mesh operator (batch.cpp:49,62 return
// TypeMismatch; SPEC.md:250 lists it as a non-goal). SURVEY.md section 8(a)
// row A17 defines the triangle-pair semantics as a composition of the
// reference's own FP64 primitives; this file is that composition and nothing
// else:
//   distance(a,b)   = min over segment_triangle_distance(e, b), e in edges(a)
//                     and segment_triangle_distance(e, a), e in edges(b)
//                     (edges are v0->v1, v1->v2, v2->v0; kernels.cpp:256)
//   intersects(a,b) = any segment_triangle_intersect over the same six
//                     (kernels.cpp:318)
//   either triangle is_degenerate() (geometry.hpp:75) => pair skipped
//   mesh result     = min over pairs p = i*|B| + j, strict '<' => lowest p
//                     (mirrors reduce_min_over_faces, kernels.cpp:359,368-376)
//   mesh intersects = lowest hit p (mirrors intersects_mesh, kernels.cpp:407)
// Row parallelism uses the reference's own for_each_chunk
// (executor.hpp:50-83) with chunk = 1 row.
#include <cstdio>
#include <cstring>
#include <string_view>
#include <variant>

#include <tindb/dataset.hpp>
#include <tindb/executor.hpp>
#include <tindb/geometry.hpp>
#include <tindb/kernels.hpp>
#include <tindb/rng.hpp>
#include <tindb/wkt.hpp>

#include "support/fixtures.hpp"

#include <atomic>
#include <cstdint>
#include <cstring>
#include <limits>
#include <vector>

using tindb::LineSegment;
using tindb::Point3;
using tindb::Triangle;
using tindb::TriangleMesh;
namespace K = tindb::kernels;

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

Triangle load_tri(const double* t) {
    return Triangle{{t[0], t[1], t[2]}, {t[3], t[4], t[5]}, {t[6], t[7], t[8]}};
}

void store_pt(double* o, const Point3& p) {
    o[0] = p.x;
    o[1] = p.y;
    o[2] = p.z;
}

// One triangle pair; witness points reported as (on a, on b).
struct PairDist {
    double d = kInf;
    Point3 on_a, on_b;
};

PairDist tri_tri_distance(const Triangle& a, const Triangle& b) {
    PairDist out;
    if (a.is_degenerate() || b.is_degenerate()) return out;
    const LineSegment ea[3] = {{a.v0, a.v1}, {a.v1, a.v2}, {a.v2, a.v0}};
    const LineSegment eb[3] = {{b.v0, b.v1}, {b.v1, b.v2}, {b.v2, b.v0}};
    for (const LineSegment& e : ea) {
        K::DistanceResult r = K::segment_triangle_distance(e, b);
        if (r.distance < out.d) {
            out.d = r.distance;
            out.on_a = r.closest_on_a;
            out.on_b = r.closest_on_b;
        }
    }
    for (const LineSegment& e : eb) {
        K::DistanceResult r = K::segment_triangle_distance(e, a);
        if (r.distance < out.d) {
            out.d = r.distance;
            out.on_a = r.closest_on_b;  // query segment lies on b here
            out.on_b = r.closest_on_a;
        }
    }
    return out;
}

bool tri_tri_intersects(const Triangle& a, const Triangle& b) {
    if (a.is_degenerate() || b.is_degenerate()) return false;
    const LineSegment ea[3] = {{a.v0, a.v1}, {a.v1, a.v2}, {a.v2, a.v0}};
    const LineSegment eb[3] = {{b.v0, b.v1}, {b.v1, b.v2}, {b.v2, b.v0}};
    for (const LineSegment& e : ea)
        if (K::segment_triangle_intersect(e, b).hit) return true;
    for (const LineSegment& e : eb)
        if (K::segment_triangle_intersect(e, a).hit) return true;
    return false;
}

std::vector<Triangle> load_mesh(const double* t, std::uint64_t n) {
    std::vector<Triangle> v(n);
    for (std::uint64_t i = 0; i < n; ++i) v[i] = load_tri(t + 9 * i);
    return v;
}

K::ExecutorConfig row_cfg(int threads) {
    return threads > 1 ? K::ExecutorConfig::parallel(threads, 1) : K::ExecutorConfig::sequential();
}

std::uint64_t copy_mesh(const TriangleMesh& m, double* out) {
    if (out) std::memcpy(out, m.triangles.data(), m.triangles.size() * sizeof(Triangle));
    return m.triangles.size();
}

}  // namespace

extern "C" {

// ---- primitives (witness layout: [dist, on_a xyz, on_b xyz]) ----
void ref_segment_segment_distance(const double* s6, const double* t6, double* out7) {
    LineSegment a{{s6[0], s6[1], s6[2]}, {s6[3], s6[4], s6[5]}};
    LineSegment b{{t6[0], t6[1], t6[2]}, {t6[3], t6[4], t6[5]}};
    K::DistanceResult r = K::segment_segment_distance(a, b);
    out7[0] = r.distance;
    store_pt(out7 + 1, r.closest_on_a);
    store_pt(out7 + 4, r.closest_on_b);
}

void ref_point_triangle_distance(const double* p3, const double* t9, double* out7) {
    K::DistanceResult r = K::point_triangle_distance({p3[0], p3[1], p3[2]}, load_tri(t9));
    out7[0] = r.distance;
    store_pt(out7 + 1, r.closest_on_a);
    store_pt(out7 + 4, r.closest_on_b);
}

void ref_segment_triangle_distance(const double* s6, const double* t9, double* out7) {
    LineSegment a{{s6[0], s6[1], s6[2]}, {s6[3], s6[4], s6[5]}};
    K::DistanceResult r = K::segment_triangle_distance(a, load_tri(t9));
    out7[0] = r.distance;
    store_pt(out7 + 1, r.closest_on_a);
    store_pt(out7 + 4, r.closest_on_b);
}

int ref_segment_triangle_intersect(const double* s6, const double* t9) {
    LineSegment a{{s6[0], s6[1], s6[2]}, {s6[3], s6[4], s6[5]}};
    return K::segment_triangle_intersect(a, load_tri(t9)).hit ? 1 : 0;
}

int ref_triangle_is_degenerate(const double* t9) { return load_tri(t9).is_degenerate() ? 1 : 0; }

// ---- triangle pairs (A17) ----
void ref_pairs_distance(const double* a9, const double* b9, std::uint64_t n, double* out7) {
    for (std::uint64_t k = 0; k < n; ++k) {
        PairDist r = tri_tri_distance(load_tri(a9 + 9 * k), load_tri(b9 + 9 * k));
        out7[7 * k] = r.d;
        store_pt(out7 + 7 * k + 1, r.on_a);
        store_pt(out7 + 7 * k + 4, r.on_b);
    }
}

void ref_pairs_intersects(const double* a9, const double* b9, std::uint64_t n, std::uint8_t* out) {
    for (std::uint64_t k = 0; k < n; ++k)
        out[k] = tri_tri_intersects(load_tri(a9 + 9 * k), load_tri(b9 + 9 * k)) ? 1 : 0;
}

// ---- mesh x mesh over rows [row_begin, row_end) step row_stride of A ----
// Returns 1 when a non-degenerate pair was seen, 0 otherwise (dist = +inf).
int ref_mesh_mesh_distance(const double* a9, std::uint64_t n, const double* b9, std::uint64_t m,
                           std::uint64_t row_begin, std::uint64_t row_end, std::uint64_t row_stride,
                           int threads, double* out7, std::uint64_t* pair_out) {
    const std::vector<Triangle> A = load_mesh(a9, n), B = load_mesh(b9, m);
    if (row_stride == 0) row_stride = 1;
    if (row_end > n) row_end = n;
    const std::uint64_t rows = row_begin < row_end ? (row_end - row_begin + row_stride - 1) / row_stride : 0;
    struct RowBest {
        PairDist r;
        std::uint64_t p = 0;
        bool found = false;
    };
    std::vector<RowBest> best(rows);
    K::for_each_chunk(row_cfg(threads), rows, [&](std::size_t, std::size_t lo, std::size_t hi) {
        for (std::size_t k = lo; k < hi; ++k) {
            const std::uint64_t i = row_begin + k * row_stride;
            RowBest rb;
            for (std::uint64_t j = 0; j < m; ++j) {
                PairDist r = tri_tri_distance(A[i], B[j]);
                if (r.d < rb.r.d) {
                    rb.r = r;
                    rb.p = i * m + j;
                    rb.found = true;
                }
            }
            best[k] = rb;
        }
    });
    RowBest out;
    for (const RowBest& rb : best)
        if (rb.found && rb.r.d < out.r.d) out = rb;
    out7[0] = out.r.d;
    store_pt(out7 + 1, out.r.on_a);
    store_pt(out7 + 4, out.r.on_b);
    *pair_out = out.found ? out.p : ~std::uint64_t(0);
    return out.found ? 1 : 0;
}

int ref_mesh_mesh_intersects(const double* a9, std::uint64_t n, const double* b9, std::uint64_t m,
                             std::uint64_t row_begin, std::uint64_t row_end, std::uint64_t row_stride,
                             int threads, std::uint64_t* pair_out) {
    const std::vector<Triangle> A = load_mesh(a9, n), B = load_mesh(b9, m);
    if (row_stride == 0) row_stride = 1;
    if (row_end > n) row_end = n;
    const std::uint64_t rows = row_begin < row_end ? (row_end - row_begin + row_stride - 1) / row_stride : 0;
    std::atomic<std::uint64_t> best{~std::uint64_t(0)};
    K::for_each_chunk(row_cfg(threads), rows, [&](std::size_t, std::size_t lo, std::size_t hi) {
        for (std::size_t k = lo; k < hi; ++k) {
            const std::uint64_t i = row_begin + k * row_stride;
            if (i * m > best.load(std::memory_order_relaxed)) return;  // cannot improve
            for (std::uint64_t j = 0; j < m; ++j) {
                if (tri_tri_intersects(A[i], B[j])) {
                    std::uint64_t p = i * m + j, seen = best.load(std::memory_order_relaxed);
                    while (p < seen && !best.compare_exchange_weak(seen, p, std::memory_order_relaxed)) {
                    }
                    break;
                }
            }
        }
    });
    *pair_out = best.load();
    return *pair_out != ~std::uint64_t(0) ? 1 : 0;
}

// ---- reference mesh generators (dataset.cpp) and fixtures (fixtures.cpp) ----
std::uint64_t ref_unit_sphere(std::uint64_t face_target, double* out) {
    return copy_mesh(tindb::bench::unit_sphere(face_target), out);
}

std::uint64_t ref_ore_body(std::uint64_t face_target, double* out) {
    tindb::bench::DatasetSpec spec;
    spec.mesh_face_target = face_target;
    return copy_mesh(tindb::bench::make_ore_body(spec), out);
}

void ref_random_triangles(std::uint64_t seed, std::uint64_t n, double lo, double hi, double* out) {
    tindb::Rng rng(seed);
    for (std::uint64_t k = 0; k < n; ++k) {
        Triangle t = tindb::fixtures::random_triangle(rng, lo, hi);
        std::memcpy(out + 9 * k, &t, sizeof(Triangle));
    }
}

// C2's terrain: the reference has no terrain generator, so
// this is the NEW heightfield restated over the reference's own Rng
// (rng.hpp:12-30, uniform(lo, hi) at :21): an nx x ny lattice over x, y in
// [0, 1000], per-vertex z = rng.uniform(-amp, amp) in row-major order, two
// CCW-up triangles per cell (v00 v10 v11, v00 v11 v01). The bench's reference
// arm builds C2 from this, never from the product library; tests pin it
// bit-for-bit to tdb_gen_terrain.
std::uint64_t ref_terrain(std::uint32_t nx, std::uint32_t ny, double amp, std::uint64_t seed, double* out) {
    const std::uint64_t faces = 2ull * nx * ny;
    if (!out || nx == 0 || ny == 0) return faces;
    tindb::Rng rng(seed);
    const std::uint64_t W = nx + 1ull;
    std::vector<Point3> v(W * (ny + 1ull));
    for (std::uint32_t iy = 0; iy <= ny; ++iy)
        for (std::uint32_t ix = 0; ix <= nx; ++ix)
            v[iy * W + ix] = Point3{1000.0 * ix / nx, 1000.0 * iy / ny, rng.uniform(-amp, amp)};
    std::uint64_t k = 0;
    auto put = [&](const Point3& a, const Point3& b, const Point3& c) {
        const Triangle t{a, b, c};
        std::memcpy(out + 9 * k++, &t, sizeof(Triangle));
    };
    for (std::uint32_t iy = 0; iy < ny; ++iy)
        for (std::uint32_t ix = 0; ix < nx; ++ix) {
            const std::uint64_t r0 = iy * W, r1 = (iy + 1ull) * W;
            put(v[r0 + ix], v[r0 + ix + 1], v[r1 + ix + 1]);
            put(v[r0 + ix], v[r1 + ix + 1], v[r1 + ix]);
        }
    return faces;
}

std::uint64_t ref_unit_cube(double* out) { return copy_mesh(tindb::fixtures::unit_cube(), out); }

// ---- segment / point x mesh: the reference's own distance_to_mesh and
// intersects_mesh (kernels.cpp:382-432) per query, record-parallel like
// run_batch (batch.cpp:94-103). face = UINT64_MAX when none.
static TriangleMesh mesh_of(const double* t9, std::uint64_t m) {
    TriangleMesh mesh;
    mesh.triangles = load_mesh(t9, m);
    mesh.refresh_degeneracy_flag();
    return mesh;
}

void ref_segments_mesh_distance(const double* s6, std::uint64_t n, const double* t9, std::uint64_t m, int threads,
                                double* dist, std::uint64_t* face) {
    const TriangleMesh mesh = mesh_of(t9, m);
    const auto inner = K::ExecutorConfig::sequential();
    K::for_each_chunk(row_cfg(threads), n, [&](std::size_t, std::size_t lo, std::size_t hi) {
        for (std::size_t k = lo; k < hi; ++k) {
            const LineSegment seg{{s6[6 * k], s6[6 * k + 1], s6[6 * k + 2]}, {s6[6 * k + 3], s6[6 * k + 4], s6[6 * k + 5]}};
            const K::DistanceResult r = K::distance_to_mesh(seg, mesh, inner);
            dist[k] = r.distance;
            face[k] = r.face_index ? *r.face_index : ~std::uint64_t(0);
        }
    });
}

void ref_points_mesh_distance(const double* p3, std::uint64_t n, const double* t9, std::uint64_t m, int threads,
                              double* dist, std::uint64_t* face) {
    const TriangleMesh mesh = mesh_of(t9, m);
    const auto inner = K::ExecutorConfig::sequential();
    K::for_each_chunk(row_cfg(threads), n, [&](std::size_t, std::size_t lo, std::size_t hi) {
        for (std::size_t k = lo; k < hi; ++k) {
            const K::DistanceResult r = K::distance_to_mesh(Point3{p3[3 * k], p3[3 * k + 1], p3[3 * k + 2]}, mesh, inner);
            dist[k] = r.distance;
            face[k] = r.face_index ? *r.face_index : ~std::uint64_t(0);
        }
    });
}

// distance_to_mesh with the mesh's has_degenerate_faces set explicitly
// (flag 0/1) instead of refreshed: the reference then evaluates (0) or skips
// (1) degenerate faces (kernels.cpp:350,357). kind 0 = segments, 1 = points.
void ref_queries_mesh_distance_flag(int kind, const double* q, std::uint64_t n, const double* t9, std::uint64_t m,
                                    int threads, int flag, double* dist, std::uint64_t* face) {
    TriangleMesh mesh;
    mesh.triangles = load_mesh(t9, m);
    mesh.has_degenerate_faces = flag != 0;
    const auto inner = K::ExecutorConfig::sequential();
    K::for_each_chunk(row_cfg(threads), n, [&](std::size_t, std::size_t lo, std::size_t hi) {
        for (std::size_t k = lo; k < hi; ++k) {
            const K::DistanceResult r =
                kind == 0 ? K::distance_to_mesh(LineSegment{{q[6 * k], q[6 * k + 1], q[6 * k + 2]},
                                                            {q[6 * k + 3], q[6 * k + 4], q[6 * k + 5]}},
                                                mesh, inner)
                          : K::distance_to_mesh(Point3{q[3 * k], q[3 * k + 1], q[3 * k + 2]}, mesh, inner);
            dist[k] = r.distance;
            face[k] = r.face_index ? *r.face_index : ~std::uint64_t(0);
        }
    });
}

void ref_segments_mesh_intersects(const double* s6, std::uint64_t n, const double* t9, std::uint64_t m, int threads,
                                  std::uint8_t* hit, std::uint64_t* face) {
    const TriangleMesh mesh = mesh_of(t9, m);
    const auto inner = K::ExecutorConfig::sequential();
    K::for_each_chunk(row_cfg(threads), n, [&](std::size_t, std::size_t lo, std::size_t hi) {
        for (std::size_t k = lo; k < hi; ++k) {
            const LineSegment seg{{s6[6 * k], s6[6 * k + 1], s6[6 * k + 2]}, {s6[6 * k + 3], s6[6 * k + 4], s6[6 * k + 5]}};
            const K::IntersectionResult r = K::intersects_mesh(seg, mesh, inner);
            hit[k] = r.hit ? 1 : 0;
            face[k] = r.face_index ? *r.face_index : ~std::uint64_t(0);
        }
    });
}

// dataset.cpp:141-165 make_drills (default box; style 0 vertical, 1 uniform)
std::uint64_t ref_make_drills(std::uint64_t seed, std::uint64_t count, int style, double* out6) {
    tindb::bench::DatasetSpec spec;
    spec.seed = seed;
    spec.segment_count = count;
    spec.drill_style = style ? tindb::bench::DrillStyle::UniformRandom : tindb::bench::DrillStyle::VerticalJittered;
    const auto d = tindb::bench::make_drills(spec);
    if (out6) std::memcpy(out6, d.data(), d.size() * sizeof(LineSegment));
    return d.size();
}

// kernels.cpp:27-46 mesh_volume (permissive policy) with a given chunk size;
// closed_out receives validate_closed (closure.cpp:41) when non-null.
double ref_mesh_volume(const double* t9, std::uint64_t n, std::uint64_t chunk, int* closed_out) {
    TriangleMesh m;
    m.triangles = load_mesh(t9, n);
    m.refresh_degeneracy_flag();
    K::ExecutorConfig cfg = K::ExecutorConfig::sequential();
    cfg.chunk_size = chunk;
    bool closed = false;
    const double v = K::mesh_volume(m, cfg, closed_out ? &closed : nullptr);
    if (closed_out) *closed_out = closed ? 1 : 0;
    return v;
}

// wkt.cpp:188 parse_wkt. Returns 0 and the geometry (kind 0 point, 1
// segment, 2 linestring, 3 mesh; coordinates in `out`, *n_out points or
// triangles; *src_out the MeshSource) or 1 with the WktParseError's what()
// and position.
int ref_parse_wkt(const char* text, std::uint64_t len, int* kind_out, double* out, std::uint64_t cap,
                  std::uint64_t* n_out, int* src_out, char* err, std::uint64_t errcap, std::uint64_t* pos_out) {
    try {
        const tindb::Geometry g = tindb::parse_wkt(std::string_view(text, len));
        *n_out = 0;
        if (auto* p = std::get_if<Point3>(&g)) {
            *kind_out = 0;
            *n_out = 1;
            if (cap >= 3) std::memcpy(out, p, sizeof *p);
        } else if (auto* sg = std::get_if<LineSegment>(&g)) {
            *kind_out = 1;
            *n_out = 2;
            if (cap >= 6) std::memcpy(out, sg, sizeof *sg);
        } else if (auto* ls = std::get_if<tindb::LineString>(&g)) {
            *kind_out = 2;
            *n_out = ls->points.size();
            if (cap >= 3 * ls->points.size()) std::memcpy(out, ls->points.data(), ls->points.size() * sizeof(Point3));
        } else if (auto* m = std::get_if<TriangleMesh>(&g)) {
            *kind_out = 3;
            *n_out = m->triangles.size();
            if (src_out) *src_out = (int)m->source_kind;
            if (cap >= 9 * m->triangles.size())
                std::memcpy(out, m->triangles.data(), m->triangles.size() * sizeof(Triangle));
        }
        return 0;
    } catch (const tindb::WktParseError& e) {
        std::snprintf(err, errcap, "%s", e.what());
        *pos_out = e.position();
        return 1;
    }
}

// wkt.cpp serialize_wkt(TriangleMesh): canonical TIN Z text, shortest
// round-trip numbers. Returns the text length (writes when it fits).
std::uint64_t ref_serialize_mesh(const double* t9, std::uint64_t n, char* out, std::uint64_t cap) {
    TriangleMesh m;
    m.triangles = load_mesh(t9, n);
    const std::string s = tindb::serialize_wkt(m);
    if (out && cap >= s.size()) std::memcpy(out, s.data(), s.size());
    return s.size();
}

}  // extern "C"
