// Bit-exact device restatement of the reference FP64 primitives.
//
// Every arithmetic operation is an explicit round-to-nearest intrinsic
// (__dadd_rn / __dsub_rn / __dmul_rn / __ddiv_rn / __dsqrt_rn), so ptxas can
// neither contract to DFMA nor reassociate: each result is the IEEE-754
// result of the same operation sequence the reference executes on x86-64
// SSE2 without FMA (proj/CMakeLists.txt Release flags).
// That makes the exact pass produce the reference's bits, which is what the
// pair index tie-break and the shortest round-trip SQL rendering
// (engine.cpp:113-117) depend on.
//
// Used only for the rare candidate pairs of the exact pass (distance) and
// for pairs that survive the conservative plane cull (intersects); the
// roofline kernel uses fast_pair.cuh.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace tdb {
namespace exact {

struct v3 {
    double x, y, z;
};

__device__ __forceinline__ v3 mk(double x, double y, double z) { return v3{x, y, z}; }
__device__ __forceinline__ v3 sub(v3 a, v3 b) {
    return mk(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y), __dsub_rn(a.z, b.z));
}
__device__ __forceinline__ v3 add(v3 a, v3 b) {
    return mk(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y), __dadd_rn(a.z, b.z));
}
__device__ __forceinline__ v3 scl(v3 a, double s) {
    return mk(__dmul_rn(a.x, s), __dmul_rn(a.y, s), __dmul_rn(a.z, s));
}
// geometry.hpp:36: (ax*bx + ay*by) + az*bz
__device__ __forceinline__ double dot(v3 a, v3 b) {
    return __dadd_rn(__dadd_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dmul_rn(a.z, b.z));
}
// geometry.hpp:38-40
__device__ __forceinline__ v3 cross(v3 a, v3 b) {
    return mk(__dsub_rn(__dmul_rn(a.y, b.z), __dmul_rn(a.z, b.y)),
              __dsub_rn(__dmul_rn(a.z, b.x), __dmul_rn(a.x, b.z)),
              __dsub_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double norm(v3 a) { return __dsqrt_rn(dot(a, a)); }
__device__ __forceinline__ bool same(v3 a, v3 b) { return a.x == b.x && a.y == b.y && a.z == b.z; }
__device__ __forceinline__ double clamp_unit(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

constexpr double kTiny = 1e-300;        // kernels.cpp:50
constexpr double kDegenArea2 = 1e-30;   // geometry.hpp:58
constexpr double kPierceEps = 1e-12;    // kernels.hpp:53
constexpr double kSlack = 1e-12;        // kernels.hpp:54

struct tri {
    v3 v0, v1, v2;
};

// geometry.hpp:75
__device__ __forceinline__ bool degenerate(const tri& t) {
    const v3 n = cross(sub(t.v1, t.v0), sub(t.v2, t.v0));
    return dot(n, n) <= kDegenArea2;
}

struct res {
    double d;
    v3 a, b;
};

// kernels::SurfaceParams (kernels.hpp:22-26), reported only when asked for
// (the per-face detail of distance_to_mesh); the hot exact passes pass null.
struct prm {
    double t, u, v;
};

// kernels.cpp:54-60
__device__ __forceinline__ res witness(v3 on_a, v3 on_b) {
    res r;
    r.a = on_a;
    r.b = on_b;
    r.d = norm(sub(on_a, on_b));
    return r;
}

// kernels.cpp:72-116
static __device__ __noinline__ res seg_seg(v3 a0, v3 a1, v3 b0, v3 b1, prm* pp = nullptr) {
    const v3 d1 = sub(a1, a0), d2 = sub(b1, b0), r = sub(a0, b0);
    const double aa = dot(d1, d1), ee = dot(d2, d2), f = dot(d2, r);
    double s = 0.0, t = 0.0;
    if (aa <= kTiny && ee <= kTiny) {
    } else if (aa <= kTiny) {
        t = clamp_unit(__ddiv_rn(f, ee));
    } else {
        const double c = dot(d1, r);
        if (ee <= kTiny) {
            s = clamp_unit(__ddiv_rn(-c, aa));
        } else {
            const double bb = dot(d1, d2);
            const double den = __dsub_rn(__dmul_rn(aa, ee), __dmul_rn(bb, bb));
            if (den > kTiny) s = clamp_unit(__ddiv_rn(__dsub_rn(__dmul_rn(bb, f), __dmul_rn(c, ee)), den));
            t = __ddiv_rn(__dadd_rn(__dmul_rn(bb, s), f), ee);
            if (t < 0.0) {
                t = 0.0;
                s = clamp_unit(__ddiv_rn(-c, aa));
            } else if (t > 1.0) {
                t = 1.0;
                s = clamp_unit(__ddiv_rn(__dsub_rn(bb, c), aa));
            }
        }
    }
    if (pp) *pp = prm{s, t, 0.0};  // kernels.cpp:110-114
    return witness(add(a0, scl(d1, s)), add(b0, scl(d2, t)));
}

// kernels.cpp:64-68, :120-124
__device__ __forceinline__ res pt_seg(v3 p, v3 s0, v3 s1) {
    const v3 d = sub(s1, s0);
    const double dd = dot(d, d);
    double t = 0.0;
    if (!(dd <= kTiny)) t = clamp_unit(__ddiv_rn(dot(sub(p, s0), d), dd));
    return witness(p, add(s0, scl(d, t)));
}

// kernels.cpp:138-227 (degenerate fallback :127-134)
static __device__ __noinline__ res pt_tri(v3 p, const tri& tr, prm* pp = nullptr) {
    const v3 e0 = sub(tr.v1, tr.v0), e1 = sub(tr.v2, tr.v0), df = sub(tr.v0, p);
    const double a00 = dot(e0, e0), a01 = dot(e0, e1), a11 = dot(e1, e1);
    const double b0 = dot(df, e0), b1 = dot(df, e1);
    const double det = __dsub_rn(__dmul_rn(a00, a11), __dmul_rn(a01, a01));
    if (degenerate(tr) || det <= kTiny) {
        res best = pt_seg(p, tr.v0, tr.v1);
        res c = pt_seg(p, tr.v0, tr.v2);
        if (c.d < best.d) best = c;
        c = pt_seg(p, tr.v1, tr.v2);
        if (c.d < best.d) best = c;
        best.a = p;
        if (pp) *pp = prm{0.0, 0.0, 0.0};  // kernels.cpp:154
        return best;
    }
    double s = __dsub_rn(__dmul_rn(a01, b1), __dmul_rn(a11, b0));
    double t = __dsub_rn(__dmul_rn(a01, b0), __dmul_rn(a00, b1));
    const double two_a01 = __dmul_rn(2.0, a01);
    if (__dadd_rn(s, t) <= det) {
        if (s < 0.0) {
            if (t < 0.0 && b0 < 0.0) {  // region 4 toward v0v1
                t = 0.0;
                s = -b0 >= a00 ? 1.0 : __ddiv_rn(-b0, a00);
            } else {  // region 4 (b0 >= 0) / region 3
                s = 0.0;
                t = b1 >= 0.0 ? 0.0 : (-b1 >= a11 ? 1.0 : __ddiv_rn(-b1, a11));
            }
        } else if (t < 0.0) {  // region 5
            t = 0.0;
            s = b0 >= 0.0 ? 0.0 : (-b0 >= a00 ? 1.0 : __ddiv_rn(-b0, a00));
        } else {  // region 0
            s = __ddiv_rn(s, det);
            t = __ddiv_rn(t, det);
        }
    } else if (s < 0.0) {  // region 2
        const double q0 = __dadd_rn(a01, b0), q1 = __dadd_rn(a11, b1);
        if (q1 > q0) {
            const double num = __dsub_rn(q1, q0), den = __dadd_rn(__dsub_rn(a00, two_a01), a11);
            s = num >= den ? 1.0 : __ddiv_rn(num, den);
            t = __dsub_rn(1.0, s);
        } else {
            s = 0.0;
            t = q1 <= 0.0 ? 1.0 : (b1 >= 0.0 ? 0.0 : __ddiv_rn(-b1, a11));
        }
    } else if (t < 0.0) {  // region 6
        const double q0 = __dadd_rn(a01, b1), q1 = __dadd_rn(a00, b0);
        if (q1 > q0) {
            const double num = __dsub_rn(q1, q0), den = __dadd_rn(__dsub_rn(a00, two_a01), a11);
            t = num >= den ? 1.0 : __ddiv_rn(num, den);
            s = __dsub_rn(1.0, t);
        } else {
            t = 0.0;
            s = q1 <= 0.0 ? 1.0 : (b0 >= 0.0 ? 0.0 : __ddiv_rn(-b0, a00));
        }
    } else {  // region 1
        const double num = __dsub_rn(__dsub_rn(__dadd_rn(a11, b1), a01), b0);
        if (num <= 0.0) {
            s = 0.0;
        } else {
            const double den = __dadd_rn(__dsub_rn(a00, two_a01), a11);
            s = num >= den ? 1.0 : __ddiv_rn(num, den);
        }
        t = __dsub_rn(1.0, s);
    }
    if (pp) *pp = prm{0.0, clamp_unit(s), clamp_unit(t)};  // kernels.cpp:221-225
    return witness(p, add(add(tr.v0, scl(e0, s)), scl(e1, t)));
}

struct pierce_t {
    bool ok;
    double t, u, v;
};

// kernels.cpp:233-252
__device__ __forceinline__ pierce_t pierce(v3 e0, v3 e1, v3 d, v3 w) {
    pierce_t r{false, 0.0, 0.0, 0.0};
    const v3 pv = cross(d, e1);
    const double den = dot(pv, e0);
    const double scale = __dmul_rn(__dmul_rn(norm(d), norm(e0)), norm(e1));
    if (fabs(den) <= __dmul_rn(kPierceEps, scale)) return r;
    const double inv = __ddiv_rn(1.0, den);
    const v3 qv = cross(w, e0);
    r.t = __dmul_rn(dot(qv, e1), inv);
    r.u = __dmul_rn(dot(pv, w), inv);
    r.v = __dmul_rn(dot(qv, d), inv);
    r.ok = true;
    return r;
}

// kernels.cpp:256-316
static __device__ __noinline__ res seg_tri(v3 p0, v3 p1, const tri& tr, prm* pp = nullptr) {
    if (same(p0, p1)) return pt_tri(p0, tr, pp);
    const v3 d = sub(p1, p0), e0 = sub(tr.v1, tr.v0), e1 = sub(tr.v2, tr.v0);
    if (!degenerate(tr)) {
        const pierce_t x = pierce(e0, e1, d, sub(p0, tr.v0));
        if (x.ok && x.u >= 0.0 && x.v >= 0.0 && __dadd_rn(x.u, x.v) <= 1.0 && x.t >= 0.0 && x.t <= 1.0) {
            if (pp) *pp = prm{x.t, x.u, x.v};  // kernels.cpp:276
            return witness(add(p0, scl(d, x.t)), add(add(tr.v0, scl(e0, x.u)), scl(e1, x.v)));
        }
    }
    res best;
    best.d = __longlong_as_double(0x7ff0000000000000LL);
    best.a = best.b = mk(0.0, 0.0, 0.0);
    prm q{0.0, 0.0, 0.0}, bp{0.0, 0.0, 0.0};
    prm* const qp = pp ? &q : nullptr;
    // edges v0v1, v0v2, v1v2 with (u, v) = (u0 + s du, v0 + s dv) (kernels.cpp:289-303)
    const double u0[3] = {0.0, 0.0, 1.0}, du[3] = {1.0, 0.0, -1.0}, dv[3] = {0.0, 1.0, 1.0};
    res c = seg_seg(p0, p1, tr.v0, tr.v1, qp);
    if (c.d < best.d) best = c, bp = prm{q.t, __dadd_rn(u0[0], __dmul_rn(q.u, du[0])), __dadd_rn(0.0, __dmul_rn(q.u, dv[0]))};
    c = seg_seg(p0, p1, tr.v0, tr.v2, qp);
    if (c.d < best.d) best = c, bp = prm{q.t, __dadd_rn(u0[1], __dmul_rn(q.u, du[1])), __dadd_rn(0.0, __dmul_rn(q.u, dv[1]))};
    c = seg_seg(p0, p1, tr.v1, tr.v2, qp);
    if (c.d < best.d) best = c, bp = prm{q.t, __dadd_rn(u0[2], __dmul_rn(q.u, du[2])), __dadd_rn(0.0, __dmul_rn(q.u, dv[2]))};
    c = pt_tri(p0, tr, qp);
    if (c.d < best.d) best = c, bp = prm{0.0, q.u, q.v};  // kernels.cpp:307-314: t = endpoint index
    c = pt_tri(p1, tr, qp);
    if (c.d < best.d) best = c, bp = prm{1.0, q.u, q.v};
    if (pp) *pp = bp;
    return best;
}

// kernels.cpp:318-336
__device__ __forceinline__ bool seg_tri_hit(v3 p0, v3 p1, const tri& tr) {
    const pierce_t x = pierce(sub(tr.v1, tr.v0), sub(tr.v2, tr.v0), sub(p1, p0), sub(p0, tr.v0));
    if (!x.ok) return false;
    if (x.t < -kSlack || x.t > 1.0 + kSlack) return false;
    if (x.u < -kSlack || x.v < -kSlack || __dadd_rn(x.u, x.v) > 1.0 + kSlack) return false;
    return true;
}

// min over the directed edges of a against b, then of b
// against a; first strict minimum wins; witnesses reported as (on a, on b).
static __device__ __noinline__ res tri_tri(const tri& a, const tri& b) {
    res best;
    best.d = __longlong_as_double(0x7ff0000000000000LL);
    best.a = best.b = mk(0.0, 0.0, 0.0);
    if (degenerate(a) || degenerate(b)) return best;
    const v3 ea[3][2] = {{a.v0, a.v1}, {a.v1, a.v2}, {a.v2, a.v0}};
    const v3 eb[3][2] = {{b.v0, b.v1}, {b.v1, b.v2}, {b.v2, b.v0}};
#pragma unroll 1
    for (int k = 0; k < 3; ++k) {
        const res c = seg_tri(ea[k][0], ea[k][1], b);
        if (c.d < best.d) best = c;
    }
#pragma unroll 1
    for (int k = 0; k < 3; ++k) {
        const res c = seg_tri(eb[k][0], eb[k][1], a);
        if (c.d < best.d) {
            best.d = c.d;
            best.a = c.b;
            best.b = c.a;
        }
    }
    return best;
}

static __device__ __noinline__ bool tri_tri_hit(const tri& a, const tri& b) {
    if (degenerate(a) || degenerate(b)) return false;
    if (seg_tri_hit(a.v0, a.v1, b) || seg_tri_hit(a.v1, a.v2, b) || seg_tri_hit(a.v2, a.v0, b))
        return true;
    return seg_tri_hit(b.v0, b.v1, a) || seg_tri_hit(b.v1, b.v2, a) || seg_tri_hit(b.v2, b.v0, a);
}

// ---- near-degenerate detection (logging only; never changes a result) -----
// A pair is near-degenerate when one of the reference's decision thresholds
// is within a factor kNearFactor of deciding it the other way:
//   * a triangle's norm2((v1-v0) x (v2-v0)) in (1e-30, 1e-30 * f^2]
//     (geometry.hpp:58,75: skipped below);
//   * a directed edge's pierce denominator |(d x e1).e0| in
//     (1e-12 s, 1e-12 s f] with s = |d||e0||e1| (kernels.cpp:243-244:
//     treated as parallel below, solved above).
constexpr double kNearFactor = 1e3;

__device__ __forceinline__ bool near_area(const tri& t) {
    const v3 n = cross(sub(t.v1, t.v0), sub(t.v2, t.v0));
    const double a2 = dot(n, n);
    return a2 > kDegenArea2 && a2 <= kDegenArea2 * kNearFactor * kNearFactor;
}

__device__ __forceinline__ bool near_parallel(v3 p0, v3 p1, const tri& t) {
    const v3 d = sub(p1, p0), e0 = sub(t.v1, t.v0), e1 = sub(t.v2, t.v0);
    const double den = fabs(dot(cross(d, e1), e0));
    const double lim = __dmul_rn(kPierceEps, __dmul_rn(__dmul_rn(norm(d), norm(e0)), norm(e1)));
    return den > lim && den <= lim * kNearFactor;
}

static __device__ __noinline__ bool near_degenerate_pair(const tri& a, const tri& b) {
    if (near_area(a) || near_area(b)) return true;
    return near_parallel(a.v0, a.v1, b) || near_parallel(a.v1, a.v2, b) || near_parallel(a.v2, a.v0, b) ||
           near_parallel(b.v0, b.v1, a) || near_parallel(b.v1, b.v2, a) || near_parallel(b.v2, b.v0, a);
}

static __device__ __noinline__ bool near_degenerate_seg(v3 p0, v3 p1, const tri& t) {
    return near_area(t) || near_parallel(p0, p1, t);
}

}  // namespace exact

// Per-call log of near-degenerate pairs (north star: "near-degenerate pairs
// logged"): a count and the first kNearLogCap (object, pair) entries.
constexpr uint32_t kNearLogCap = 1024;
struct NearLog {
    unsigned long long* count;
    unsigned long long* entries;  // 2 per entry: object, pair
    unsigned long long base = 0;  // the count's value when the call began (a counter that is never reset)
};

__device__ __forceinline__ void near_log(const NearLog& L, unsigned long long obj, unsigned long long pair) {
    if (!L.count) return;
    const unsigned long long k = atomicAdd(L.count, 1ull) - L.base;
    if (k < kNearLogCap) {
        L.entries[2 * k] = obj;
        L.entries[2 * k + 1] = pair;
    }
}
}  // namespace tdb
