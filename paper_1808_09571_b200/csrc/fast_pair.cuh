// FP64 triangle-pair filter — the roofline device code.
//
// For a non-intersecting pair the exact distance is attained by one of
//   * 9 edge/edge pairs (clamped segment-segment, Ericson's two-sided clamp:
//     s from the unconstrained solve, t optimal for s, s optimal for the
//     clamped t — covers vertex/edge and vertex/vertex contacts too), and
//   * 6 vertex/face pairs (vertex projecting inside the other triangle).
// Intersecting pairs are caught by a plane-straddle test followed by a
// division-free piercing test (rare branch, out of line). Everything is
// squared distances with FMA; the only reciprocal is rcp.approx
// (MUFU.RCP64H) + one Newton step for the first s (the value is always a
// distance between two real points of the triangles; its excess over the
// true distance is bounded in DESIGN.md 4.2). No DDIV/DSQRT. Cost per
// candidate (FP64 pipe): vertex/face 12, a face's three A vertices + the
// straddle signs 51, an edge of B against A's three edges 90.
//
// The value d~^2 approximates the A17 composition's distance
// closely enough to bound it: the exact pass (distance.cu) re-evaluates with
// the bit-exact composition every pair whose d~ lies inside a band around the
// minimum.
#pragma once

#include <cuda_runtime.h>

#include "tdb_internal.h"

namespace tdb {

__device__ __forceinline__ double pos_inf() { return __longlong_as_double(0x7ff0000000000000LL); }

// clamp to [0,1] with integer ops only (keeps the FP64 pipe free):
// negative (incl. -0, -NaN) -> 0, >= 1 (incl. +inf, +NaN) -> 1.
__device__ __forceinline__ double clamp01(double x) {
    int hi = __double2hiint(x), lo = __double2loint(x);
    const int neg = hi >> 31;
    hi &= ~neg;
    lo &= ~neg;
    const bool ge1 = hi >= 0x3ff00000;
    return __hiloint2double(ge1 ? 0x3ff00000 : hi, ge1 ? 0 : lo);
}

// min of two non-negative doubles (or +inf) as ordered 64-bit integers.
__device__ __forceinline__ double min_nn(double a, double b) {
    return __double_as_longlong(a) < __double_as_longlong(b) ? a : b;
}

__device__ __forceinline__ double rcp_approx(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    return r;
}

// eta(m) of tdb_internal.h: L = max edge, kmax = max F_K, ext = max |coord|
__device__ __forceinline__ double band_eta_of(double L, double kmax, double ext, double m) {
    const double w = m + 4.0 * L;
    return kBandEdge * sqrt(L * w) + kmax * w + kBandAbs * ext;
}

// 1/x to ~2^-40 relative: rcp.approx (MUFU.RCP64H, ~2^-20) plus one Newton
// step (2 DFMA). Drops the first-parameter error of the edge/edge solve from
// first order in 2^-20 to the cancellation floor of its num / den
// (DESIGN.md 4.2).
__device__ __forceinline__ double rcp_nr(double x) {
    const double r = rcp_approx(x);
    return fma(r, fma(-x, r, 1.0), r);
}

__device__ __forceinline__ bool all_nonneg(double a, double b, double c) {
    return (__double2hiint(a) | __double2hiint(b) | __double2hiint(c)) >= 0;
}

// Field access: field f of a face lives at p[f * stride] (SoA planes in HBM:
// stride = n_pad; staged sub-tile in SMEM: stride = kSB; AoS record: 1).
struct FaceRef {
    const double* p;
    uint64_t stride;
    __device__ __forceinline__ double operator()(int f) const { return p[(uint64_t)f * stride]; }
};

struct FaceRefLdg {
    const double* p;
    uint64_t stride;
    __device__ __forceinline__ double operator()(int f) const { return __ldg(p + (uint64_t)f * stride); }
};

// A-side face held in registers for the whole B chunk.
struct AFace {
    double v[9];   // vertices
    double e[9];   // cyclic edges
    double L[3];   // |E|^2
    double IL[3];  // 1/|E|^2
    double n[3];   // unit normal
    double U[3], W[3];
};

template <class P>
__device__ __forceinline__ void load_aface(AFace& A, const P& at) {
#pragma unroll
    for (int k = 0; k < 9; ++k) A.v[k] = at(F_V + k);
#pragma unroll
    for (int k = 0; k < 9; ++k) A.e[k] = at(F_E + k);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        A.L[k] = at(F_L + k);
        A.IL[k] = at(F_IL + k);
        A.n[k] = at(F_N + k);
        A.U[k] = at(F_U + k);
        A.W[k] = at(F_W + k);
    }
}

__device__ __forceinline__ double dot3(const double* a, double x, double y, double z) {
    return fma(a[0], x, fma(a[1], y, a[2] * z));
}

// Division-free piercing test: does an edge of the triangle with vertex
// heights h (w.r.t. the other's plane) and barycentrics (u, v) cross the
// other triangle? Crossing of edge k->k+1 at lambda = h_k/(h_k - h_k+1);
// u(X)*(h_k - h_k+1) = h_k u_k+1 - h_k+1 u_k, likewise for v and 1 - u - v.
__device__ __forceinline__ bool edges_pierce(const double h[3], const double u[3], const double v[3]) {
    bool hit = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int q = k == 2 ? 0 : k + 1;
        const double D = h[k] - h[q];
        if ((__double2hiint(h[k]) ^ __double2hiint(h[q])) < 0 && D != 0.0) {
            const double uD = fma(h[k], u[q], -h[q] * u[k]);
            const double vD = fma(h[k], v[q], -h[q] * v[k]);
            const double tD = D - uD - vD;
            hit |= D > 0.0 ? (uD >= 0.0 && vD >= 0.0 && tD >= 0.0) : (uD <= 0.0 && vD <= 0.0 && tD <= 0.0);
        }
    }
    return hit;
}

// B's face as the filter stages it (tdb_internal.h): its face-vertices record
// (V at FV_V) and its face-planes record (N, U, W at FP_N, FP_U, FP_W), read
// through the plane field numbers F_V / F_N / F_U / F_W.
struct FaceRec {
    const double* fv;
    const double* fp;
    __device__ __forceinline__ double operator()(int f) const {
        return f < F_E ? fv[FV_V + f] : f < F_U ? fp[FP_N + f - F_N] : f < F_W ? fp[FP_U + f - F_U] : fp[FP_W + f - F_W];
    }
};

// Out-of-line (rare) piercing test for a pair whose triangles both straddle
// the other's plane; reloads both faces so the hot path keeps no state.
template <class PB>
static __device__ __noinline__ bool pierce_t(const double* ap, uint64_t as, PB B) {
    const FaceRef A{ap, as};
    double hb[3], ub[3], vb[3], ha[3], ua[3], va[3];
    const double a0x = A(F_V), a0y = A(F_V + 1), a0z = A(F_V + 2);
    const double b0x = B(F_V), b0y = B(F_V + 1), b0z = B(F_V + 2);
    const double na[3] = {A(F_N), A(F_N + 1), A(F_N + 2)}, nb[3] = {B(F_N), B(F_N + 1), B(F_N + 2)};
    const double Ua[3] = {A(F_U), A(F_U + 1), A(F_U + 2)}, Ub[3] = {B(F_U), B(F_U + 1), B(F_U + 2)};
    const double Wa[3] = {A(F_W), A(F_W + 1), A(F_W + 2)}, Wb[3] = {B(F_W), B(F_W + 1), B(F_W + 2)};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double wx = B(F_V + 3 * k) - a0x, wy = B(F_V + 3 * k + 1) - a0y, wz = B(F_V + 3 * k + 2) - a0z;
        hb[k] = dot3(na, wx, wy, wz);
        ub[k] = dot3(Ua, wx, wy, wz);
        vb[k] = dot3(Wa, wx, wy, wz);
        const double qx = A(F_V + 3 * k) - b0x, qy = A(F_V + 3 * k + 1) - b0y, qz = A(F_V + 3 * k + 2) - b0z;
        ha[k] = dot3(nb, qx, qy, qz);
        ua[k] = dot3(Ub, qx, qy, qz);
        va[k] = dot3(Wb, qx, qy, qz);
    }
    return edges_pierce(hb, ub, vb) || edges_pierce(ha, ua, va);
}

static __device__ __forceinline__ bool pierce_slow(const double* ap, uint64_t as, const double* bp, uint64_t bs) {
    return pierce_t(ap, as, FaceRef{bp, bs});
}

constexpr int kInfHi = 0x7ff00000;  // high word of +inf


// Barycentric inside test u >= 0, v >= 0, u + v < 1 with one FP64 add: the
// sum is non-negative when u, v are, so "< 1" is a high-word compare
// (u + v in [1, 1 + 2^-20) reads as outside: a boundary case the edge/edge
// candidates cover exactly).
__device__ __forceinline__ bool inside(double u, double v) {
    return ((__double2hiint(u) | __double2hiint(v)) >= 0) & (__double2hiint(u + v) < 0x3ff00000);
}

// ---- the candidate families -------------------------------
// Minima are kept as the high 32 bits of non-negative doubles (a lower bound
// within a relative 2^-20 of the value: one VIMNMX per candidate).

// Vertex P of B against face A: |h| when P projects inside A (w = P - A_0);
// hs = the high word of h (its sign says which side of A's plane P is on).
__device__ __forceinline__ int vertex_cand(const AFace& A, double px, double py, double pz, int& hs) {
    const double wx = px - A.v[0], wy = py - A.v[1], wz = pz - A.v[2];
    const double h = dot3(A.n, wx, wy, wz);
    const double u = dot3(A.U, wx, wy, wz);
    const double v = dot3(A.W, wx, wy, wz);
    hs = __double2hiint(h);
    return inside(u, v) ? (hs & 0x7fffffff) : kInfHi;
}

// The vertices of A against face B (vertex B_0, unit normal nb, dual basis
// ub / vb): |h| when inside, min into hmin. Returns true when A straddles B's
// plane; w0 = A_0 - B_0.
__device__ __forceinline__ bool a_vertex_cand(const AFace& A, double b0x, double b0y, double b0z, const double nb[3],
                                              const double ub[3], const double vb[3], int& hmin, double w0[3]) {
    int ha_or = 0, ha_and = -1;
#pragma unroll
    for (int j = 0; j < 3; ++j) {  // A_j - B_0
        const double wx = A.v[3 * j] - b0x, wy = A.v[3 * j + 1] - b0y, wz = A.v[3 * j + 2] - b0z;
        if (j == 0) w0[0] = wx, w0[1] = wy, w0[2] = wz;
        const double h = dot3(nb, wx, wy, wz);
        const double u = dot3(ub, wx, wy, wz);
        const double v = dot3(vb, wx, wy, wz);
        ha_or |= __double2hiint(h);
        ha_and &= __double2hiint(h);
        hmin = min(hmin, inside(u, v) ? (__double2hiint(h) & 0x7fffffff) : kInfHi);
    }
    return !(ha_or >= 0 || ha_and < 0);
}

// B's vertices b[9] straddle A's plane (sign words of their heights; B_0's
// from w0 = A_0 - B_0: B_0 - A_0 = -w0 exactly).
__device__ __forceinline__ bool b_straddles(const AFace& A, const double b[9], const double w0[3]) {
    const double h0 = -dot3(A.n, w0[0], w0[1], w0[2]);
    const double h1 = dot3(A.n, b[3] - A.v[0], b[4] - A.v[1], b[5] - A.v[2]);
    const double h2 = dot3(A.n, b[6] - A.v[0], b[7] - A.v[1], b[8] - A.v[2]);
    const int hb_or = __double2hiint(h0) | __double2hiint(h1) | __double2hiint(h2);
    const int hb_and = __double2hiint(h0) & __double2hiint(h1) & __double2hiint(h2);
    return !(hb_or >= 0 || hb_and < 0);
}

// Edge Q -> Q + Ea of A (|Ea|^2 = La, 1/|Ea|^2 = ILa) against edge P -> P + Eb
// of B: Ericson's clamped segment distance, squared, high word (s from the
// unconstrained solve with a Newton-refined reciprocal, t optimal for s, s
// optimal for the clamped t; every value is the distance between two real
// points of the segments).
__device__ __forceinline__ int edge_pair(double qx, double qy, double qz, double eax, double eay, double eaz,
                                         double La, double ILa, double px, double py, double pz, double ebx,
                                         double eby, double ebz, double Lb, double ILb) {
    const double wx = px - qx, wy = py - qy, wz = pz - qz;  // w = P - Q
    const double fw = fma(ebx, wx, fma(eby, wy, ebz * wz));
    const double bb = fma(eax, ebx, fma(eay, eby, eaz * ebz));
    const double cw = fma(eax, wx, fma(eay, wy, eaz * wz));
    // s0 = (cw Lb - bb fw) / (La Lb - bb^2), both terms divided by Lb
    const double bbI = bb * ILb;
    const double den = fma(-bbI, bb, La);
    const double num = fma(-bbI, fw, cw);
    double s = clamp01(num * rcp_nr(den));
    const double t = clamp01(fma(bb, s, -fw) * ILb);
    s = clamp01(fma(bb, t, cw) * ILa);
    const double dx = fma(s, eax, fma(-t, ebx, -wx));
    const double dy = fma(s, eay, fma(-t, eby, -wy));
    const double dz = fma(s, eaz, fma(-t, ebz, -wz));
    return __double2hiint(fma(dx, dx, fma(dy, dy, dz * dz)));
}

// ---- FP32 edge/edge candidate (FULL mode's shared edge lists, DESIGN.md 4.1/4.2)
// The same clamped solve as edge_pair on FP32 copies of the edges, with both
// start points relative to one origin o (B's box centre): Q' = fl(Q - o),
// P' = fl(P - o), E = fl(E), |E|^2, 1/|E|^2 rounded once. Every value is
// still the distance between two points of (float-rounded) edges; its excess
// over the true edge/edge distance is bounded by eta_f32 (below). The FP64
// exact pass is unchanged: this only decides which items it re-scans.
__device__ __forceinline__ float rcp_approx_f32(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// A edge: Q' (3), E (3), |E|^2, 1/|E|^2; B edge record p0 = P'x P'y P'z Ebx,
// p1 = Eby Ebz Lb ILb. Returns d~^2.
__device__ __forceinline__ float edge_pair32(const float (&q)[8], float4 p0, float4 p1) {
    const float wx = p0.x - q[0], wy = p0.y - q[1], wz = p0.z - q[2];  // w = P - Q
    const float fw = fmaf(p0.w, wx, fmaf(p1.x, wy, p1.y * wz));
    const float bb = fmaf(q[3], p0.w, fmaf(q[4], p1.x, q[5] * p1.y));
    const float cw = fmaf(q[3], wx, fmaf(q[4], wy, q[5] * wz));
    const float bbI = bb * p1.w;
    const float den = fmaf(-bbI, bb, q[6]);
    const float num = fmaf(-bbI, fw, cw);
    float s = __saturatef(num * rcp_approx_f32(den));  // NaN -> 0: any s in [0, 1] is a point of the edge
    const float t = __saturatef(fmaf(bb, s, -fw) * p1.w);
    s = __saturatef(fmaf(bb, t, cw) * q[7]);
    const float dx = fmaf(s, q[3], fmaf(-t, p0.w, -wx));
    const float dy = fmaf(s, q[4], fmaf(-t, p1.x, -wy));
    const float dz = fmaf(s, q[5], fmaf(-t, p1.y, -wz));
    return fmaf(dx, dx, fmaf(dy, dy, dz * dz));
}

// The same candidate for two A edges at once on packed FP32 pairs
// (fma/mul/sub .rn.f32x2, SASS FFMA2/FMUL2/FADD2): lane k of every packed
// operation is the IEEE operation edge_pair32 performs for A edge k, or its
// exact negation (x * -y = -(x * y), fma(a, -b, c) = c - a b, rounded
// alike), so each half returns edge_pair32's value bit for bit and eta_f32
// is unchanged. B's components enter as {x, x} broadcasts (ptxas folds them
// into the FFMA2 scalar operand). Q2[k] = {A edge 0's field k, A edge 1's};
// Q2[3..5] are passed negated (nE = -E_A) beside E_A itself.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2f(float a, float b) {
    f32x2 d;
    asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(a), "f"(b));
    return d;
}
__device__ __forceinline__ float lo_f(f32x2 x) { return __uint_as_float((unsigned)x); }
__device__ __forceinline__ float hi_f(f32x2 x) { return __uint_as_float((unsigned)(x >> 32)); }
__device__ __forceinline__ f32x2 fma2f(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f32x2 mul2f(f32x2 a, f32x2 b) {
    f32x2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f32x2 sub2f(f32x2 a, f32x2 b) {
    f32x2 d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

struct AEdge32x2 {
    f32x2 q[3];   // Q' (start point about o)
    f32x2 e[3];   // E_A
    f32x2 ne[3];  // -E_A
    f32x2 L;      // |E_A|^2
    float il[2];  // 1/|E_A|^2
};

// B edge record p0 = P'x P'y P'z Ebx, p1 = Eby Ebz Lb ILb (nILb = -ILb).
// Returns {d~^2 for A edge 0, for A edge 1}.
__device__ __forceinline__ void edge_pair32x2(const AEdge32x2& A, float4 p0, float4 p1, float nILb, float& d0,
                                              float& d1) {
    const f32x2 Px = pk2f(p0.x, p0.x), Py = pk2f(p0.y, p0.y), Pz = pk2f(p0.z, p0.z);
    const f32x2 Ex = pk2f(p0.w, p0.w), Ey = pk2f(p1.x, p1.x), Ez = pk2f(p1.y, p1.y);
    const f32x2 nIL = pk2f(nILb, nILb);
    const f32x2 wx = sub2f(Px, A.q[0]), wy = sub2f(Py, A.q[1]), wz = sub2f(Pz, A.q[2]);  // w = P - Q
    const f32x2 fw = fma2f(Ex, wx, fma2f(Ey, wy, mul2f(Ez, wz)));
    const f32x2 bb = fma2f(A.e[0], Ex, fma2f(A.e[1], Ey, mul2f(A.e[2], Ez)));
    const f32x2 cw = fma2f(A.e[0], wx, fma2f(A.e[1], wy, mul2f(A.e[2], wz)));
    const f32x2 nbbI = mul2f(bb, nIL);                       // -(bb * ILb)
    const f32x2 den = fma2f(nbbI, bb, A.L);                  // fmaf(-bbI, bb, |E_A|^2)
    const f32x2 num = fma2f(nbbI, fw, cw);                   // fmaf(-bbI, fw, cw)
    const float s0 = __saturatef(lo_f(num) * rcp_approx_f32(lo_f(den)));
    const float s1 = __saturatef(hi_f(num) * rcp_approx_f32(hi_f(den)));
    const f32x2 nfw = mul2f(fw, pk2f(-1.0f, -1.0f));         // exact
    const f32x2 tp = fma2f(bb, pk2f(s0, s1), nfw);           // fmaf(bb, s, -fw)
    const float t0 = __saturatef(lo_f(tp) * p1.w), t1 = __saturatef(hi_f(tp) * p1.w);
    const f32x2 t = pk2f(t0, t1);
    const f32x2 sp = fma2f(bb, t, cw);                       // fmaf(bb, t, cw)
    const f32x2 s = pk2f(__saturatef(lo_f(sp) * A.il[0]), __saturatef(hi_f(sp) * A.il[1]));
    // -d: -dx = fmaf(s, -q3, fmaf(t, Ebx, wx)) (fmaf(-t, Ebx, -wx) negated)
    const f32x2 dx = fma2f(s, A.ne[0], fma2f(t, Ex, wx));
    const f32x2 dy = fma2f(s, A.ne[1], fma2f(t, Ey, wy));
    const f32x2 dz = fma2f(s, A.ne[2], fma2f(t, Ez, wz));
    const f32x2 d2 = fma2f(dx, dx, fma2f(dy, dy, mul2f(dz, dz)));
    d0 = lo_f(d2);
    d1 = hi_f(d2);
}

// A non-negative float as the double of the same value, by integer ops
// (no F2F): the item minima are non-negative doubles compared as u64.
__device__ __forceinline__ unsigned long long f32_as_f64_bits(float x) {
    const unsigned u = __float_as_uint(x);
    if (u == 0u) return 0ull;
    if (u >= 0x7f800000u) return 0x7ff0000000000000ull;  // +inf (NaN never reaches here: fminf drops it)
    if (u < 0x00800000u) return (unsigned long long)__double_as_longlong((double)x);  // subnormal (rare)
    return ((unsigned long long)((u >> 3) + 0x38000000u) << 32) | ((unsigned long long)(u << 29));
}

// eta of the FP32 edge/edge candidate, added to eta(m) when the FP32 lists
// ran. u = 2^-24; L = max edge; rB = B's box half-diagonal.
//   solve: squared excess X = 12 u L (|w| + L) <= kF32Solve L (m + 4L): the
//          excess in d is <= min(sqrt X, X / 2d) (sqrt(d^2 + X) - d);
//   data:  the float start points / edges / w and the evaluation move the
//          point pair by <= u (2 rB + 10 (m + 4L)).
// Margins 4x. The sqrt / (X / 2d) pair is not monotone in d, so the value
// used is its supremum over d <= m: max(4 min(sqrt X, X / 2m), 4.5 sqrt X - m).
constexpr double kF32Solve = 12.0 * 5.9604644775390625e-8;
constexpr double kF32Lin = 4.0 * 10.0 * 5.9604644775390625e-8;
constexpr double kF32Org = 4.0 * 2.0 * 5.9604644775390625e-8;
__device__ __forceinline__ double eta_f32(double L, double rB, double m) {
    const double w = m + 4.0 * L;
    const double X = kF32Solve * L * w, sx = sqrt(X);
    const double solve = m > 0.5 * sx ? X / (2.0 * m) : sx;
    return fmax(4.0 * solve, 4.5 * sx - m) + kF32Lin * w + kF32Org * rB;
}

// Edge P -> P + Eb of B (|Eb|^2 = Lb, 1/|Eb|^2 = ILb) against A's three edges.
__device__ __forceinline__ int edge_cand(const AFace& A, double px, double py, double pz, double ebx, double eby,
                                         double ebz, double Lb, double ILb) {
    int c[3];
#pragma unroll
    for (int j = 0; j < 3; ++j)
        c[j] = edge_pair(A.v[3 * j], A.v[3 * j + 1], A.v[3 * j + 2], A.e[3 * j], A.e[3 * j + 1], A.e[3 * j + 2],
                         A.L[j], A.IL[j], px, py, pz, ebx, eby, ebz, Lb, ILb);
    return min(min(c[0], c[1]), c[2]);
}

// The smallest |h| high word (hmin) as the high word of h^2.
__device__ __forceinline__ int hmin_sq(int hmin) {
    const double hv = __hiloint2double(hmin, 0);  // truncated |h|
    return __double2hiint(hv * hv);
}

// d~^2 of the pair (face A in registers, face B through `bt`, plane layout),
// truncated to its high word: the minimum of the pair's 15 candidates
// (vertex_cand x 3, a_vertex_cand's 3, edge_cand x 3), 0 when an edge pierces a
// face. The filter kernel evaluates the same candidates, each shared vertex
// and edge once per feature block (distance.cu). `ap`/`as` locate A's fields
// for the out-of-line piercing test.
// kEdges = false leaves out the edge/edge candidates (tdb_pairs_filter_f32
// adds them in FP32, as FULL mode does).
template <class P, bool kEdges = true>
__device__ __forceinline__ double pair_d2(const AFace& A, const P& bt, const double* ap, uint64_t as) {
    double b[9], nb[3], ub[3], vb[3];
#pragma unroll
    for (int k = 0; k < 9; ++k) b[k] = bt(F_V + k);
#pragma unroll
    for (int k = 0; k < 3; ++k) nb[k] = bt(F_N + k), ub[k] = bt(F_U + k), vb[k] = bt(F_W + k);
    int hmin = kInfHi, best = kInfHi, hs;
    double w0[3];
    bool straddle = a_vertex_cand(A, b[0], b[1], b[2], nb, ub, vb, hmin, w0);
    straddle = straddle && b_straddles(A, b, w0);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        hmin = min(hmin, vertex_cand(A, b[3 * k], b[3 * k + 1], b[3 * k + 2], hs));
        if (kEdges)
            best = min(best, edge_cand(A, b[3 * k], b[3 * k + 1], b[3 * k + 2], bt(F_E + 3 * k), bt(F_E + 3 * k + 1),
                                   bt(F_E + 3 * k + 2), bt(F_L + k), bt(F_IL + k)));
    }
    best = min(best, hmin_sq(hmin));
    if (straddle && pierce_slow(ap, as, bt.p, bt.stride)) best = 0;
    return __hiloint2double(best, 0);
}


}  // namespace tdb
