// Drives include/tindb_b200/kernels.hpp against the REFERENCE's own types
// and dispatch (compiled with -Dtindb=tindb_ref and linked with
// oracle/_ref/libtindb_ref.so, i.e. the unmodified reference sources).
// Run by tests/test_gpu_shim.py on a B200; prints "SHIM OK".
#include <tindb/batch.hpp>
#include <tindb/dataset.hpp>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdint>

#include "tindb_b200/kernels.hpp"

extern "C" int ref_mesh_mesh_distance(const double*, std::uint64_t, const double*, std::uint64_t,
                                      std::uint64_t, std::uint64_t, std::uint64_t, int, double*,
                                      std::uint64_t*);
extern "C" int ref_mesh_mesh_intersects(const double*, std::uint64_t, const double*, std::uint64_t,
                                        std::uint64_t, std::uint64_t, std::uint64_t, int,
                                        std::uint64_t*);

using namespace tindb;
namespace K = tindb::kernels;

static int fails = 0;
#define EXPECT(c)                                                        \
    do {                                                                 \
        if (!(c)) {                                                      \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);     \
            ++fails;                                                     \
        }                                                                \
    } while (0)

static TriangleMesh shifted(const TriangleMesh& m, double dx, double dy, double dz, double s = 1.0) {
    TriangleMesh o = m;
    for (Triangle& t : o.triangles)
        for (Point3* p : {&t.v0, &t.v1, &t.v2}) *p = Point3{p->x * s + dx, p->y * s + dy, p->z * s + dz};
    return o;
}

static const double* F(const TriangleMesh& m) { return reinterpret_cast<const double*>(m.triangles.data()); }

static bool same_bits(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }

int main() {
    const TriangleMesh s = bench::unit_sphere(1000);
    const TriangleMesh far = shifted(s, 2.5, 0, 0);
    const TriangleMesh cross = shifted(s, 0.5, 0.1, 0);
    auto cfg = K::ExecutorConfig::parallel(4);

    // mesh_mesh_distance vs the reference composition (A17)
    for (const TriangleMesh* b : {&far, &cross}) {
        K::b200::MeshPairInfo info;
        K::DistanceResult r = K::b200::mesh_mesh_distance(s, *b, cfg, &info);
        double o7[7];
        std::uint64_t p = 0;
        ref_mesh_mesh_distance(F(s), s.triangles.size(), F(*b), b->triangles.size(), 0, s.triangles.size(), 1,
                               4, o7, &p);
        EXPECT(same_bits(r.distance, o7[0]));
        EXPECT(info.pair_index && *info.pair_index == p);
        EXPECT(r.face_index && *r.face_index == p / b->triangles.size());
        EXPECT(same_bits(r.closest_on_a.x, o7[1]) && same_bits(r.closest_on_b.z, o7[6]));
        std::uint64_t hp = 0;
        const int hit = ref_mesh_mesh_intersects(F(s), s.triangles.size(), F(*b), b->triangles.size(), 0,
                                                 s.triangles.size(), 1, 4, &hp);
        K::IntersectionResult h = K::b200::mesh_mesh_intersects(s, *b, cfg, &info);
        EXPECT(h.hit == (hit != 0));
        if (h.hit) EXPECT(info.pair_index && *info.pair_index == hp);
    }

    // the same through a device group (every device of the box)
    {
        K::b200::DeviceGroup g;
        for (const TriangleMesh* b : {&far, &cross}) {
            K::b200::MeshPairInfo i1, i2;
            K::DistanceResult r1 = K::b200::mesh_mesh_distance(s, *b, cfg, &i1);
            K::DistanceResult r2 = K::b200::mesh_mesh_distance(g, s, *b, &i2);
            EXPECT(same_bits(r1.distance, r2.distance) && i1.pair_index == i2.pair_index);
            EXPECT(same_bits(r1.closest_on_b.y, r2.closest_on_b.y));
            K::IntersectionResult h1 = K::b200::mesh_mesh_intersects(s, *b, cfg, &i1);
            K::IntersectionResult h2 = K::b200::mesh_mesh_intersects(g, s, *b, &i2);
            EXPECT(h1.hit == h2.hit && i1.pair_index == i2.pair_index);
        }
    }

    // the missing batch.cpp:49/:62 branch
    EXPECT(!K::b200::eval_mesh_mesh(K::BatchOp::Distance, Geometry{LineSegment{{0, 0, 0}, {1, 1, 1}}},
                                    Geometry{s}, cfg));
    auto v = K::b200::eval_mesh_mesh(K::BatchOp::Distance, Geometry{s}, Geometry{far}, cfg);
    EXPECT(v && std::holds_alternative<double>(*v) && std::get<double>(*v) == 0.5);

    // whole-column run_batch: meshes on the device, everything else through
    // the reference dispatch, results in record order with record ids
    std::vector<store::GeometryRecord> recs;
    recs.push_back({11, Geometry{shifted(s, 0.3, 0, 0, 0.5)}});
    recs.push_back({12, Geometry{LineSegment{{3, 0, 0}, {4, 0, 0}}}});
    recs.push_back({13, Geometry{shifted(s, -3.0, 1.0, 0, 0.2)}});
    recs.push_back({14, Geometry{Point3{0, 0, 5}}});
    recs.push_back({15, Geometry{LineString{{{0, 0, 0}, {1, 0, 0}, {1, 1, 0}}}}});
    recs.push_back({16, Geometry{LineSegment{{-2, -2, -2}, {2, 2, 2}}}});        // pierces the sphere
    recs.push_back({17, Geometry{LineSegment{{0.1, 0.1, 0.1}, {0.1, 0.1, 0.1}}}});  // zero length
    recs.push_back({18, Geometry{LineString{{{1.5, 0, 0}, {2, 0, 0}}}}});       // 2-point line string
    recs.push_back({19, Geometry{Point3{0.2, 0.1, 0.3}}});
    {  // a drill column in the sphere's frame
        bench::DatasetSpec spec;
        spec.segment_count = 300;
        for (const LineSegment& d : bench::make_drills(spec)) {
            const Point3 a{d.p0.x / 400.0 - 1.25, d.p0.y / 400.0 - 1.25, d.p0.z / 200.0 + 1.0};
            const Point3 b{d.p1.x / 400.0 - 1.25, d.p1.y / 400.0 - 1.25, d.p1.z / 200.0 + 1.0};
            recs.push_back({100 + (std::int64_t)recs.size(), Geometry{LineSegment{a, b}}});
        }
    }
    const std::optional<Geometry> lit = Geometry{s};
    for (K::BatchOp op : {K::BatchOp::Distance, K::BatchOp::Intersects}) {
        auto got = K::b200::run_batch_b200(op, recs, lit, cfg);
        auto ref = K::run_batch(op, recs, lit, cfg);  // TypeMismatch for Mesh x Mesh
        EXPECT(got.size() == recs.size());
        for (std::size_t i = 0; i < recs.size(); ++i) {
            EXPECT(got[i].record_id == recs[i].id);
            if (kind_of(recs[i].geometry) == GeometryKind::Mesh) {
                EXPECT(ref[i].is_error());
                const auto& m = std::get<TriangleMesh>(recs[i].geometry);
                if (op == K::BatchOp::Distance) {
                    double o7[7];
                    std::uint64_t p = 0;
                    ref_mesh_mesh_distance(F(m), m.triangles.size(), F(s), s.triangles.size(), 0,
                                           m.triangles.size(), 1, 4, o7, &p);
                    EXPECT(std::holds_alternative<double>(got[i].value) &&
                           same_bits(std::get<double>(got[i].value), o7[0]));
                } else {
                    std::uint64_t hp = 0;
                    const int hit = ref_mesh_mesh_intersects(F(m), m.triangles.size(), F(s), s.triangles.size(),
                                                             0, m.triangles.size(), 1, 4, &hp);
                    EXPECT(std::holds_alternative<bool>(got[i].value) && std::get<bool>(got[i].value) == (hit != 0));
                }
            } else {
                EXPECT(got[i].value.index() == ref[i].value.index());
                if (std::holds_alternative<double>(ref[i].value))
                    EXPECT(same_bits(std::get<double>(got[i].value), std::get<double>(ref[i].value)));
                if (std::holds_alternative<bool>(ref[i].value))
                    EXPECT(std::get<bool>(got[i].value) == std::get<bool>(ref[i].value));
            }
        }
    }
    // distance_to_mesh / intersects_mesh: every field of the reference's
    // result (distance, face, closest points, params; hit, point, params),
    // bit for bit, over segments and points near a sphere mesh (with
    // crossings, grazing and zero-length segments)
    {
        const TriangleMesh m = shifted(bench::unit_sphere(2000), 0.25, -0.5, 0.125);
        std::uint64_t st = 12345;
        auto rnd = [&st] {  // xorshift in [-1.5, 1.5)
            st ^= st << 13, st ^= st >> 7, st ^= st << 17;
            return (double)(st >> 11) * 0x1.0p-53 * 3.0 - 1.5;
        };
        int hits = 0;
        for (int k = 0; k < 400; ++k) {
            const Point3 p0{rnd(), rnd(), rnd()};
            const Point3 p1 = k % 10 == 0 ? p0 : Point3{rnd(), rnd(), rnd()};
            const LineSegment seg{p0, p1};
            auto cmp = [&](const K::DistanceResult& a, const K::DistanceResult& b) {
                EXPECT(same_bits(a.distance, b.distance) && a.face_index == b.face_index);
                EXPECT(same_bits(a.closest_on_a.x, b.closest_on_a.x) && same_bits(a.closest_on_a.y, b.closest_on_a.y) &&
                       same_bits(a.closest_on_a.z, b.closest_on_a.z));
                EXPECT(same_bits(a.closest_on_b.x, b.closest_on_b.x) && same_bits(a.closest_on_b.y, b.closest_on_b.y) &&
                       same_bits(a.closest_on_b.z, b.closest_on_b.z));
                EXPECT(a.params.has_value() == b.params.has_value());
                if (a.params && b.params)
                    EXPECT(same_bits(a.params->t, b.params->t) && same_bits(a.params->u, b.params->u) &&
                           same_bits(a.params->v, b.params->v));
            };
            cmp(K::b200::distance_to_mesh(seg, m, cfg), K::distance_to_mesh(seg, m, cfg));
            cmp(K::b200::distance_to_mesh(p0, m, cfg), K::distance_to_mesh(p0, m, cfg));
            const K::IntersectionResult hd = K::b200::intersects_mesh(seg, m, cfg);
            const K::IntersectionResult hr = K::intersects_mesh(seg, m, cfg);
            EXPECT(hd.hit == hr.hit && hd.face_index == hr.face_index && hd.point.has_value() == hr.point.has_value());
            if (hd.point && hr.point)
                EXPECT(same_bits(hd.point->x, hr.point->x) && same_bits(hd.point->y, hr.point->y) &&
                       same_bits(hd.point->z, hr.point->z));
            if (hd.params && hr.params)
                EXPECT(same_bits(hd.params->t, hr.params->t) && same_bits(hd.params->u, hr.params->u) &&
                       same_bits(hd.params->v, hr.params->v) && same_bits(hd.params->w, hr.params->w));
            hits += hr.hit;
        }
        EXPECT(hits > 20 && hits < 380);
        bool threw = false;
        try {
            K::b200::distance_to_mesh(Geometry{m}, m, cfg);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        EXPECT(threw);
    }

    // has_degenerate_faces is honoured as the reference reads it
    // (kernels.cpp:350,357): test_distance.cpp:278-290's mesh, without and with
    // refresh_degeneracy_flag()
    {
        TriangleMesh m;
        m.triangles.push_back(Triangle{{0, 0, 1}, {1, 0, 1}, {2, 0, 1}});  // degenerate, closer
        m.triangles.push_back(Triangle{{0, 0, 0}, {1, 0, 0}, {0, 1, 0}});
        for (int refresh = 0; refresh < 2; ++refresh) {
            if (refresh) m.refresh_degeneracy_flag();
            const Point3 p{0.2, 0.1, 2.0};
            const LineSegment seg{{0.2, 0.1, 2.0}, {0.3, 0.2, 1.5}};
            const K::DistanceResult a = K::b200::distance_to_mesh(p, m, cfg), b = K::distance_to_mesh(p, m, cfg);
            EXPECT(same_bits(a.distance, b.distance) && a.face_index == b.face_index);
            EXPECT(a.face_index && *a.face_index == (refresh ? 1u : 0u));
            const K::DistanceResult c = K::b200::distance_to_mesh(seg, m, cfg), d = K::distance_to_mesh(seg, m, cfg);
            EXPECT(same_bits(c.distance, d.distance) && c.face_index == d.face_index);
            // run_batch: a Point literal over a Mesh column (batch.cpp:44-48)
            std::vector<store::GeometryRecord> recs{{7, Geometry{m}}, {8, Geometry{shifted(m, 0, 0, 0.5)}}};
            const auto rb = K::b200::run_batch_b200(K::BatchOp::Distance, recs, Geometry{p}, cfg);
            const auto rr = K::run_batch(K::BatchOp::Distance, recs, Geometry{p}, cfg);
            for (int k = 0; k < 2; ++k)
                EXPECT(same_bits(std::get<double>(rb[k].value), std::get<double>(rr[k].value)));
        }
    }

    // the device mesh cache: same content -> one upload, any change -> a new entry
    {
        auto& cache = K::b200::default_mesh_cache();
        cache.clear();
        const TriangleMesh m = bench::unit_sphere(1000);
        const Point3 p{0.3, -0.2, 1.7};
        const auto r1 = K::b200::distance_to_mesh(p, m, cfg);
        const auto r2 = K::b200::distance_to_mesh(p, TriangleMesh(m), cfg);  // equal copy: a hit
        EXPECT(cache.size() == 1 && same_bits(r1.distance, r2.distance) && r1.face_index == r2.face_index);
        TriangleMesh moved = m;
        moved.triangles[5].v1.x = std::nextafter(moved.triangles[5].v1.x, 2.0);
        const auto r3 = K::b200::distance_to_mesh(p, moved, cfg);
        EXPECT(cache.size() == 2);
        const auto r4 = K::distance_to_mesh(p, moved, cfg);
        EXPECT(same_bits(r3.distance, r4.distance) && r3.face_index == r4.face_index);
    }

    if (fails == 0) std::printf("SHIM OK\n");
    return fails ? 1 : 0;
}
