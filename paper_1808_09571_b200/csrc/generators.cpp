// Host mesh generators — the synthetic side of the "mesh/geometry loader".
//
// unit_sphere / ore_body restate the reference generator
// (/root/reference/proj/src/dataset.cpp:28-139): a regular octahedron or
// icosahedron, subdivided k times with normalised edge midpoints, chosen so
// the face count 8*4^a or 20*4^b is nearest the target (ties prefer the
// icosahedron). Every face is emitted as a 72-byte triangle in face order,
// so the output is bit-identical to the reference's TriangleMesh (pinned by
// tests/test_generators.py against oracle/_ref).
//
// terrain is NEW (the reference has no terrain): an nx x ny lattice over
// x, y in [0, 1000] with per-vertex z ~ U(-amp, amp) drawn from
// mt19937_64(seed) through the reference's portable uniform mapping
// (rng.hpp:12-30), two CCW-up triangles per cell.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <unordered_map>
#include <vector>

#include "tindb_b200.h"

namespace {

struct P3 {
    double x, y, z;
};

P3 unit(const P3& p) {
    const double n = std::sqrt(p.x * p.x + p.y * p.y + p.z * p.z);
    return {p.x / n, p.y / n, p.z / n};
}

struct Poly {
    std::vector<P3> v;
    std::vector<std::array<uint32_t, 3>> f;
};

Poly octahedron() {
    Poly m;
    m.v = {{1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1}};
    m.f = {{0, 2, 4}, {2, 1, 4}, {1, 3, 4}, {3, 0, 4}, {2, 0, 5}, {1, 2, 5}, {3, 1, 5}, {0, 3, 5}};
    return m;
}

Poly icosahedron() {
    const double g = (1.0 + std::sqrt(5.0)) / 2.0;
    Poly m;
    m.v = {{-1, g, 0}, {1, g, 0}, {-1, -g, 0}, {1, -g, 0}, {0, -1, g}, {0, 1, g},
           {0, -1, -g}, {0, 1, -g}, {g, 0, -1}, {g, 0, 1}, {-g, 0, -1}, {-g, 0, 1}};
    for (P3& p : m.v) p = unit(p);
    m.f = {{0, 11, 5}, {0, 5, 1},  {0, 1, 7},   {0, 7, 10}, {0, 10, 11}, {1, 5, 9},  {5, 11, 4},
           {11, 10, 2}, {10, 7, 6}, {7, 1, 8},  {3, 9, 4},  {3, 4, 2},   {3, 2, 6},  {3, 6, 8},
           {3, 8, 9},  {4, 9, 5},  {2, 4, 11}, {6, 2, 10}, {8, 6, 7},   {9, 8, 1}};
    return m;
}

// One 4:1 split. Midpoints are shared through an edge-keyed cache so that
// neighbouring faces reference bitwise-identical vertices (watertight).
void split(Poly& m) {
    std::unordered_map<uint64_t, uint32_t> mid;
    mid.reserve(m.f.size() * 2);
    auto midpoint = [&](uint32_t a, uint32_t b) {
        const uint64_t key = (uint64_t(std::min(a, b)) << 32) | std::max(a, b);
        auto it = mid.find(key);
        if (it != mid.end()) return it->second;
        const P3 &pa = m.v[a], &pb = m.v[b];
        const P3 s{(pa.x + pb.x) * 0.5, (pa.y + pb.y) * 0.5, (pa.z + pb.z) * 0.5};
        const uint32_t idx = uint32_t(m.v.size());
        m.v.push_back(unit(s));
        mid.emplace(key, idx);
        return idx;
    };
    std::vector<std::array<uint32_t, 3>> out;
    out.reserve(m.f.size() * 4);
    for (const auto& t : m.f) {
        const uint32_t ab = midpoint(t[0], t[1]);
        const uint32_t bc = midpoint(t[1], t[2]);
        const uint32_t ca = midpoint(t[2], t[0]);
        out.push_back({t[0], ab, ca});
        out.push_back({t[1], bc, ab});
        out.push_back({t[2], ca, bc});
        out.push_back({ab, bc, ca});
    }
    m.f.swap(out);
}

struct Choice {
    bool ico;
    int level;
    uint64_t faces;
};

// dataset.cpp:85-102
Choice pick(uint64_t target) {
    auto gap = [target](uint64_t c) { return c > target ? c - target : target - c; };
    Choice best{true, 0, 20};
    for (int ico = 1; ico >= 0; --ico) {
        const uint64_t base = ico ? 20 : 8;
        for (int level = 0; level < 12; ++level) {
            const uint64_t faces = base << (2 * level);
            const bool better =
                gap(faces) < gap(best.faces) || (gap(faces) == gap(best.faces) && ico && !best.ico);
            if (better) best = {ico != 0, level, faces};
            if (faces > target * 4) break;
        }
    }
    return best;
}

Poly sphere(uint64_t target, uint64_t* faces) {
    const Choice c = pick(target);
    *faces = c.faces;
    Poly m = c.ico ? icosahedron() : octahedron();
    for (int k = 0; k < c.level; ++k) split(m);
    return m;
}

void emit(const Poly& m, double* out) {
    for (size_t i = 0; i < m.f.size(); ++i)
        for (int c = 0; c < 3; ++c) {
            const P3& p = m.v[m.f[i][c]];
            out[9 * i + 3 * c + 0] = p.x;
            out[9 * i + 3 * c + 1] = p.y;
            out[9 * i + 3 * c + 2] = p.z;
        }
}

}  // namespace

extern "C" uint64_t tdb_gen_unit_sphere(uint64_t face_target, double* out) {
    if (!out) return pick(face_target).faces;
    uint64_t faces = 0;
    emit(sphere(face_target, &faces), out);
    return faces;
}

// dataset.cpp:125-139: the box is x,y in [0,1000], z in [-400,0]
// (dataset.hpp:15-21); radius = 0.3 * min extent, centre = box centre, and
// the vertex array is transformed before faces are emitted.
extern "C" uint64_t tdb_gen_ore_body(uint64_t face_target, double* out) {
    if (!out) return pick(face_target).faces;
    uint64_t faces = 0;
    Poly m = sphere(face_target, &faces);
    const P3 lo{0.0, 0.0, -400.0}, hi{1000.0, 1000.0, 0.0};
    const P3 ext{hi.x - lo.x, hi.y - lo.y, hi.z - lo.z};
    const double radius = 0.3 * std::min({ext.x, ext.y, ext.z});
    const P3 ctr{(lo.x + hi.x) * 0.5, (lo.y + hi.y) * 0.5, (lo.z + hi.z) * 0.5};
    for (P3& p : m.v) p = {ctr.x + p.x * radius, ctr.y + p.y * radius, ctr.z + p.z * radius};
    emit(m, out);
    return faces;
}

// dataset.cpp:141-165 make_drills over the default DatasetSpec box; style 0 =
// VerticalJittered (collar on the top face, tilted hole), 1 = UniformRandom.
// Same mt19937_64 stream and the same draw order as the reference.
extern "C" uint64_t tdb_gen_drills(uint64_t seed, uint64_t count, int style, double* out6) {
    if (!out6) return count;
    std::mt19937_64 eng(seed);
    auto uniform = [&](double lo, double hi) { return lo + (hi - lo) * (double(eng() >> 11) * 0x1.0p-53); };
    const P3 lo{0.0, 0.0, -400.0}, hi{1000.0, 1000.0, 0.0};
    for (uint64_t i = 0; i < count; ++i) {
        double* o = out6 + 6 * i;
        if (style == 1) {
            for (int e = 0; e < 2; ++e) {
                o[3 * e] = uniform(lo.x, hi.x);
                o[3 * e + 1] = uniform(lo.y, hi.y);
                o[3 * e + 2] = uniform(lo.z, hi.z);
            }
            continue;
        }
        const double cx = uniform(lo.x, hi.x);
        const double cy = uniform(lo.y, hi.y);
        const double cz = hi.z;
        const double depth = uniform(0.4, 1.0) * (hi.z - lo.z);
        const double tx = uniform(-0.15, 0.15);
        const double ty = uniform(-0.15, 0.15);
        o[0] = cx, o[1] = cy, o[2] = cz;
        o[3] = cx + tx * depth, o[4] = cy + ty * depth, o[5] = cz - depth;
    }
    return count;
}

extern "C" uint64_t tdb_gen_terrain(uint32_t nx, uint32_t ny, double amp, uint64_t seed,
                                    double* out) {
    const uint64_t faces = 2ull * nx * ny;
    if (!out || nx == 0 || ny == 0) return faces;
    std::mt19937_64 eng(seed);
    auto uniform = [&](double lo, double hi) {
        const double u = double(eng() >> 11) * 0x1.0p-53;
        return lo + (hi - lo) * u;
    };
    const uint32_t W = nx + 1;
    std::vector<P3> v(size_t(W) * (ny + 1));
    for (uint32_t iy = 0; iy <= ny; ++iy)
        for (uint32_t ix = 0; ix <= nx; ++ix)
            v[size_t(iy) * W + ix] = {1000.0 * ix / nx, 1000.0 * iy / ny, uniform(-amp, amp)};
    size_t k = 0;
    auto put = [&](const P3& a, const P3& b, const P3& c) {
        const P3* q[3] = {&a, &b, &c};
        for (int t = 0; t < 3; ++t) {
            out[9 * k + 3 * t] = q[t]->x;
            out[9 * k + 3 * t + 1] = q[t]->y;
            out[9 * k + 3 * t + 2] = q[t]->z;
        }
        ++k;
    };
    for (uint32_t iy = 0; iy < ny; ++iy)
        for (uint32_t ix = 0; ix < nx; ++ix) {
            const P3& v00 = v[size_t(iy) * W + ix];
            const P3& v10 = v[size_t(iy) * W + ix + 1];
            const P3& v11 = v[size_t(iy + 1) * W + ix + 1];
            const P3& v01 = v[size_t(iy + 1) * W + ix];
            put(v00, v10, v11);
            put(v00, v11, v01);
        }
    return faces;
}
