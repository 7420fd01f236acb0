// tindb_b200 C++ shim: the Mesh x Mesh operators on the reference's own
// operator surface (tindb::kernels, /root/reference/proj/include/tindb/
// kernels.hpp and batch.hpp), backed by the sm_100a engine through the C ABI
// (tindb_b200.h). Header-only; drop it next to the reference sources and
// link libtindb_b200.so.
//
// * mesh_mesh_distance / mesh_mesh_intersects — new kernels:: entries beside
//   distance_to_mesh / intersects_mesh (kernels.hpp:68-90). Results use the
//   reference result types: face_index = the face of `a`; the pair index and
//   the face of `b` are reported through MeshPairInfo.
// * eval_mesh_mesh — the branch batch.cpp:49 (eval_distance) and :62
//   (eval_intersects) lack today; returns nullopt for other pairings so the
//   reference's dispatch continues unchanged.
// * run_batch_b200 — run_batch (batch.hpp:49-51) against a Mesh literal with
//   the Mesh records (triangle pairs), the Segment / 2-point LineString
//   records and the Point records (distance_to_mesh / intersects_mesh, the
//   paper's drill workload) each evaluated as one device column; every other
//   pairing is delegated to the reference run_batch, in record order.
//
// Error behaviour mirrors the reference: invalid input throws
// std::invalid_argument (kernels.cpp:403), device failures throw
// std::runtime_error; pairing errors stay TypeMismatch values and never
// throw out of run_batch_b200 (batch.hpp:17-22).
#pragma once

#include <tindb/batch.hpp>
#include <tindb/geometry.hpp>
#include <tindb/kernels.hpp>
#include <tindb/store_types.hpp>

#include <cstdint>
#include <limits>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include "tindb_b200.h"

namespace tindb::kernels::b200 {

static_assert(sizeof(Triangle) == 9 * sizeof(double), "TriangleMesh must be 72-byte AoS faces");

inline void check(int rc) {
    if (rc == TDB_OK) return;
    const std::string msg = tdb_last_error();
    if (rc == TDB_E_ARG) throw std::invalid_argument(msg);
    throw std::runtime_error("tindb_b200: " + msg);
}

inline const double* faces_of(const TriangleMesh& m) {
    return reinterpret_cast<const double*>(m.triangles.data());
}

// A device-resident copy of an immutable mesh (TableSnapshot meshes are
// immutable once Ready, store_types.hpp:21-32, so copies may be cached).
class DeviceMesh {
  public:
    explicit DeviceMesh(const TriangleMesh& m) {
        check(tdb_mesh_upload(faces_of(m), m.triangles.size(), &h_));
        faces_ = m.triangles.size();
    }
    ~DeviceMesh() { tdb_mesh_free(h_); }
    DeviceMesh(const DeviceMesh&) = delete;
    DeviceMesh& operator=(const DeviceMesh&) = delete;
    tdb_mesh handle() const { return h_; }
    std::size_t faces() const { return faces_; }

  private:
    tdb_mesh h_ = nullptr;
    std::size_t faces_ = 0;
};

struct MeshPairInfo {
    std::optional<std::uint64_t> pair_index;  // i * |b| + j, lowest on ties
    std::optional<std::size_t> face_a, face_b;
};

inline DistanceResult mesh_mesh_distance(const DeviceMesh& a, const DeviceMesh& b,
                                         MeshPairInfo* info = nullptr) {
    tdb_dist_out o{};
    check(tdb_mesh_mesh_distance(a.handle(), b.handle(), &o));
    DistanceResult r;
    r.distance = o.distance;
    if (o.found) {
        r.closest_on_a = {o.on_a[0], o.on_a[1], o.on_a[2]};
        r.closest_on_b = {o.on_b[0], o.on_b[1], o.on_b[2]};
        r.face_index = static_cast<std::size_t>(o.i);
    }
    if (info) {
        *info = {};
        if (o.found) info->pair_index = o.pair, info->face_a = o.i, info->face_b = o.j;
    }
    return r;
}

// ST_3DDistance(a, b) over every triangle pair. `cfg` is
// accepted for signature parity with distance_to_mesh; the device decides
// its own parallelism.
inline DistanceResult mesh_mesh_distance(const TriangleMesh& a, const TriangleMesh& b,
                                         const ExecutorConfig& /*cfg*/ = ExecutorConfig::sequential(),
                                         MeshPairInfo* info = nullptr) {
    DeviceMesh da(a), db(b);
    return mesh_mesh_distance(da, db, info);
}

inline IntersectionResult mesh_mesh_intersects(const DeviceMesh& a, const DeviceMesh& b,
                                               MeshPairInfo* info = nullptr) {
    tdb_hit_out o{};
    check(tdb_mesh_mesh_intersects(a.handle(), b.handle(), &o));
    IntersectionResult r;
    r.hit = o.hit != 0;
    if (r.hit) r.face_index = static_cast<std::size_t>(o.i);
    if (info) {
        *info = {};
        if (r.hit) info->pair_index = o.pair, info->face_a = o.i, info->face_b = o.j;
    }
    return r;
}

inline IntersectionResult mesh_mesh_intersects(const TriangleMesh& a, const TriangleMesh& b,
                                               const ExecutorConfig& /*cfg*/ = ExecutorConfig::sequential(),
                                               MeshPairInfo* info = nullptr) {
    DeviceMesh da(a), db(b);
    return mesh_mesh_intersects(da, db, info);
}

// The missing Mesh x Mesh branch of eval_distance / eval_intersects
// (batch.cpp:31-63); nullopt for any other pairing.
inline std::optional<KernelValue> eval_mesh_mesh(BatchOp op, const Geometry& record, const Geometry& arg,
                                                 const ExecutorConfig& cfg) {
    if (kind_of(record) != GeometryKind::Mesh || kind_of(arg) != GeometryKind::Mesh) return std::nullopt;
    const auto& a = std::get<TriangleMesh>(record);
    const auto& b = std::get<TriangleMesh>(arg);
    if (op == BatchOp::Distance) return KernelValue{mesh_mesh_distance(a, b, cfg).distance};
    if (op == BatchOp::Intersects) return KernelValue{mesh_mesh_intersects(a, b, cfg).hit};
    return std::nullopt;
}

// run_batch (batch.hpp:49-51) with the Mesh column on the device: one upload
// of the column (CSR face offsets + per-object AABB headers), one launch.
inline std::vector<KernelResult> run_batch_b200(BatchOp op, const std::vector<store::GeometryRecord>& records,
                                                const std::optional<Geometry>& argument,
                                                const ExecutorConfig& cfg) {
    const bool mesh_arg = argument && kind_of(*argument) == GeometryKind::Mesh;
    if (!mesh_arg || (op != BatchOp::Distance && op != BatchOp::Intersects))
        return run_batch(op, records, argument, cfg);

    std::vector<KernelResult> out(records.size());
    std::vector<std::size_t> mesh_rows, seg_rows, pt_rows, other_rows;
    for (std::size_t i = 0; i < records.size(); ++i) {
        const GeometryKind k = kind_of(records[i].geometry);
        if (k == GeometryKind::Mesh) mesh_rows.push_back(i);
        else if (k == GeometryKind::Segment) seg_rows.push_back(i);  // incl. 2-point line strings
        else if (k == GeometryKind::Point && op == BatchOp::Distance) pt_rows.push_back(i);
        else other_rows.push_back(i);
    }
    // Segment / Point x Mesh (batch.cpp:37-40, :58): distance_to_mesh /
    // intersects_mesh per record, the whole column in one device call
    if (!seg_rows.empty() || !pt_rows.empty()) {
        DeviceMesh lit(std::get<TriangleMesh>(*argument));
        auto run_queries = [&](const std::vector<std::size_t>& rows, int kind) {
            if (rows.empty()) return;
            const int width = kind == TDB_QUERY_SEGMENTS ? 6 : 3;
            std::vector<double> q(width * rows.size());
            for (std::size_t k = 0; k < rows.size(); ++k) {
                const Geometry& g = records[rows[k]].geometry;
                if (kind == TDB_QUERY_SEGMENTS) {
                    const LineSegment s = segment_view(g);
                    const double v[6] = {s.p0.x, s.p0.y, s.p0.z, s.p1.x, s.p1.y, s.p1.z};
                    std::copy(v, v + 6, q.begin() + 6 * k);
                } else {
                    const Point3& p = std::get<Point3>(g);
                    q[3 * k] = p.x, q[3 * k + 1] = p.y, q[3 * k + 2] = p.z;
                }
            }
            tdb_queries qs = nullptr;
            check(tdb_queries_upload(q.data(), rows.size(), kind, &qs));
            struct FreeQ {
                tdb_queries q;
                ~FreeQ() { tdb_queries_free(q); }
            } gq{qs};
            std::vector<double> dist(rows.size());
            std::vector<std::uint8_t> hit(rows.size());
            std::vector<std::uint64_t> face(rows.size());
            if (op == BatchOp::Distance)
                check(tdb_queries_mesh_distance(qs, lit.handle(), dist.data(), face.data()));
            else
                check(tdb_queries_mesh_intersects(qs, lit.handle(), hit.data(), face.data()));
            for (std::size_t k = 0; k < rows.size(); ++k) {
                KernelResult& r = out[rows[k]];
                r.record_id = records[rows[k]].id;
                if (op == BatchOp::Distance) r.value = dist[k];
                else r.value = hit[k] != 0;
            }
        };
        run_queries(seg_rows, TDB_QUERY_SEGMENTS);
        run_queries(pt_rows, TDB_QUERY_POINTS);
    }

    if (!other_rows.empty()) {  // reference dispatch for every other pairing
        std::vector<store::GeometryRecord> rest;
        rest.reserve(other_rows.size());
        for (std::size_t i : other_rows) rest.push_back(records[i]);
        std::vector<KernelResult> r = run_batch(op, rest, argument, cfg);
        for (std::size_t k = 0; k < other_rows.size(); ++k) out[other_rows[k]] = std::move(r[k]);
    }
    if (mesh_rows.empty()) return out;

    std::vector<std::uint64_t> off(mesh_rows.size() + 1, 0);
    for (std::size_t k = 0; k < mesh_rows.size(); ++k)
        off[k + 1] = off[k] + std::get<TriangleMesh>(records[mesh_rows[k]].geometry).triangles.size();
    std::vector<double> faces(9 * off.back());
    for (std::size_t k = 0; k < mesh_rows.size(); ++k) {
        const auto& m = std::get<TriangleMesh>(records[mesh_rows[k]].geometry);
        std::copy(faces_of(m), faces_of(m) + 9 * m.triangles.size(), faces.begin() + 9 * off[k]);
    }
    tdb_table t = nullptr;
    check(tdb_table_upload(faces.data(), off.data(), mesh_rows.size(), &t));
    struct Free {
        tdb_table t;
        ~Free() { tdb_table_free(t); }
    } guard{t};
    DeviceMesh lit(std::get<TriangleMesh>(*argument));
    std::vector<double> dist(mesh_rows.size());
    std::vector<std::uint8_t> hit(mesh_rows.size());
    if (op == BatchOp::Distance)
        check(tdb_table_eval(TDB_OP_DISTANCE, t, lit.handle(), dist.data(), nullptr, nullptr));
    else
        check(tdb_table_eval(TDB_OP_INTERSECTS, t, lit.handle(), nullptr, hit.data(), nullptr));
    for (std::size_t k = 0; k < mesh_rows.size(); ++k) {
        KernelResult& r = out[mesh_rows[k]];
        r.record_id = records[mesh_rows[k]].id;
        if (op == BatchOp::Distance) r.value = dist[k];
        else r.value = hit[k] != 0;
    }
    return out;
}

}  // namespace tindb::kernels::b200
