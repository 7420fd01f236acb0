// FP64 triangle-pair filter — the roofline device code.
//
// For a non-intersecting pair the exact distance is attained by one of
//   * 9 edge/edge pairs (clamped segment-segment, Ericson's two-sided clamp:
//     s from the unconstrained solve, t optimal for s, s optimal for the
//     clamped t — covers vertex/edge and vertex/vertex contacts too), and
//   * 6 vertex/face pairs (vertex projecting inside the other triangle).
// Intersecting pairs are caught by a plane-straddle test followed by a
// division-free piercing test (rare branch). Everything is squared distances
// with FMA; the only reciprocal is rcp.approx (MUFU.RCP64H) for the first s,
// which only perturbs the evaluated point pair to second order (the value is
// always a distance between two real points of the triangles). Per pair:
// 27 DADD (vertex differences) + 6 x 12 (vertex/face) + 9 x 27 (edge/edge)
// = 342 FP64 pipe instructions, no DDIV/DSQRT.
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

__device__ __forceinline__ bool all_nonneg(double a, double b, double c) {
    return (__double2hiint(a) | __double2hiint(b) | __double2hiint(c)) >= 0;
}

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

// Division-free piercing test (rare branch): does an edge of one triangle
// cross the other? Heights h (signed, scaled) and barycentrics (u, v) of the
// three vertices of the piercing triangle w.r.t. the pierced one. Crossing of
// edge k->k+1 at lambda = h_k/(h_k - h_k+1); u(X)*(h_k - h_k+1) =
// h_k u_k+1 - h_k+1 u_k, likewise for v and for 1 - u - v.
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
            const bool pos = D > 0.0;
            hit |= pos ? (uD >= 0.0 && vD >= 0.0 && tD >= 0.0) : (uD <= 0.0 && vD <= 0.0 && tD <= 0.0);
        }
    }
    return hit;
}

// d~^2 for face A (registers) against face j of the B accessor.
// `bt(f)` returns field f of the B face.
template <class P>
__device__ __forceinline__ double pair_d2(const AFace& A, const P& bt) {
    double best = pos_inf();
    double hb[3], ha[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double bx = bt(F_V + 3 * k), by = bt(F_V + 3 * k + 1), bz = bt(F_V + 3 * k + 2);
        double w[3][3];  // w_j = B_k - A_j
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            w[j][0] = bx - A.v[3 * j];
            w[j][1] = by - A.v[3 * j + 1];
            w[j][2] = bz - A.v[3 * j + 2];
        }
        {  // vertex B_k against face A
            const double h = dot3(A.n, w[0][0], w[0][1], w[0][2]);
            const double u = dot3(A.U, w[0][0], w[0][1], w[0][2]);
            const double v = dot3(A.W, w[0][0], w[0][1], w[0][2]);
            const double t = (1.0 - u) - v;
            hb[k] = h;
            best = min_nn(best, all_nonneg(u, v, t) ? h * h : pos_inf());
        }
        if (k == 0) {  // vertices A_j against face B: A_j - B_0 = -w_j
            const double nb[3] = {bt(F_N), bt(F_N + 1), bt(F_N + 2)};
            const double ub[3] = {bt(F_U), bt(F_U + 1), bt(F_U + 2)};
            const double vb[3] = {bt(F_W), bt(F_W + 1), bt(F_W + 2)};
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const double h = dot3(nb, w[j][0], w[j][1], w[j][2]);
                const double u = -dot3(ub, w[j][0], w[j][1], w[j][2]);
                const double v = -dot3(vb, w[j][0], w[j][1], w[j][2]);
                const double t = (1.0 - u) - v;
                ha[j] = h;
                best = min_nn(best, all_nonneg(u, v, t) ? h * h : pos_inf());
            }
        }
        const double ebx = bt(F_E + 3 * k), eby = bt(F_E + 3 * k + 1), ebz = bt(F_E + 3 * k + 2);
        const double Lb = bt(F_L + k), ILb = bt(F_IL + k);
#pragma unroll
        for (int j = 0; j < 3; ++j) {  // edge A_j->A_j+1 against edge B_k->B_k+1
            const double* ea = A.e + 3 * j;
            const double cw = dot3(ea, w[j][0], w[j][1], w[j][2]);
            const double fw = fma(ebx, w[j][0], fma(eby, w[j][1], ebz * w[j][2]));
            const double bb = dot3(ea, ebx, eby, ebz);
            const double den = fma(-bb, bb, A.L[j] * Lb);
            const double num = fma(cw, Lb, -(bb * fw));
            double s = clamp01(num * rcp_approx(den));
            const double t = clamp01(fma(bb, s, -fw) * ILb);
            s = clamp01(fma(bb, t, cw) * A.IL[j]);
            const double dx = fma(s, ea[0], fma(-t, ebx, -w[j][0]));
            const double dy = fma(s, ea[1], fma(-t, eby, -w[j][1]));
            const double dz = fma(s, ea[2], fma(-t, ebz, -w[j][2]));
            best = min_nn(best, fma(dx, dx, fma(dy, dy, dz * dz)));
        }
    }
    // Both triangles straddle the other's plane: an edge may pierce a face.
    const bool sa = !(all_nonneg(hb[0], hb[1], hb[2]) || ((__double2hiint(hb[0]) & __double2hiint(hb[1]) & __double2hiint(hb[2])) < 0));
    const bool sb = !(all_nonneg(ha[0], ha[1], ha[2]) || ((__double2hiint(ha[0]) & __double2hiint(ha[1]) & __double2hiint(ha[2])) < 0));
    if (sa && sb) {
        double u[3], v[3], u2[3], v2[3];
        const double nb[3] = {bt(F_N), bt(F_N + 1), bt(F_N + 2)};
        const double ub[3] = {bt(F_U), bt(F_U + 1), bt(F_U + 2)};
        const double vb[3] = {bt(F_W), bt(F_W + 1), bt(F_W + 2)};
        const double b0x = bt(F_V), b0y = bt(F_V + 1), b0z = bt(F_V + 2);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double wx = bt(F_V + 3 * k) - A.v[0], wy = bt(F_V + 3 * k + 1) - A.v[1],
                         wz = bt(F_V + 3 * k + 2) - A.v[2];
            u[k] = dot3(A.U, wx, wy, wz);
            v[k] = dot3(A.W, wx, wy, wz);
            const double qx = A.v[3 * k] - b0x, qy = A.v[3 * k + 1] - b0y, qz = A.v[3 * k + 2] - b0z;
            u2[k] = dot3(ub, qx, qy, qz);
            v2[k] = dot3(vb, qx, qy, qz);
        }
        (void)nb;
        if (edges_pierce(hb, u, v) || edges_pierce(ha, u2, v2)) best = 0.0;
    }
    return best;
}

}  // namespace tdb
