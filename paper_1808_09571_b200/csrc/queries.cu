// Segment x mesh and point x mesh: the paper's own workload (drill holes vs
// an ore body) on the same device store and the same
// filter -> exact-pass design as the triangle pairs.
//
// Semantics are the reference's, per query (batch.cpp:31-63 -> kernels.cpp):
//   distance   distance_to_mesh(seg|point, mesh) (kernels.cpp:382-405):
//              min over non-degenerate faces (kernels.cpp:350-357) of
//              segment_triangle_distance / point_triangle_distance, lowest
//              face index on ties; a zero-length segment is a point query
//              (kernels.cpp:388-391)
//   intersects intersects_mesh(seg, mesh) (kernels.cpp:407-432): the lowest
//              face whose segment_triangle_intersect hits (every face is
//              tested, degenerate ones through the exact predicate)
//
// Layout: queries are uploaded per call into SoA planes; a CTA holds 128
// queries (one per thread) and streams a B chunk through shared memory with
// TMA bulk copies. Filter values are high-word truncated squared distances
// (fast_pair.cuh conventions); the exact pass re-evaluates, with the
// bit-exact reference primitives (exact.cuh), every (query, face) whose
// filter value lies inside the query's band.
#include <algorithm>
#include <cstring>
#include <vector>

#include "exact.cuh"
#include "runtime.h"
#include "tma.cuh"

namespace tdb {

namespace {

constexpr unsigned long long kNone = ~0ull;
enum { QK_SEG = 0, QK_POINT = 1 };

struct QArgs {
    const double* Q;  // query planes: 6 (segments: p0 xyz, p1 xyz) or 3 (points), stride Qpad
    uint64_t Qn, Qpad;
    int kind;
    const double* Bp;
    uint64_t Bn_pad, Bn, n_chunks, chunk;
    double* itemmin;
    unsigned long long* qmin;
};

// ---- filter values -----------------------------------------------------------
// point P vs face B: vertex/face projection + the three clamped point/edge
// distances.
template <class P>
__device__ __forceinline__ int pt_d2(double px, double py, double pz, const P& bt) {
    const double qx = px - bt(F_V), qy = py - bt(F_V + 1), qz = pz - bt(F_V + 2);
    int best = kInfHi, hmin = kInfHi;
    {
        const double nb[3] = {bt(F_N), bt(F_N + 1), bt(F_N + 2)};
        const double ub[3] = {bt(F_U), bt(F_U + 1), bt(F_U + 2)};
        const double vb[3] = {bt(F_W), bt(F_W + 1), bt(F_W + 2)};
        const double h = dot3(nb, qx, qy, qz), u = dot3(ub, qx, qy, qz), v = dot3(vb, qx, qy, qz);
        hmin = inside(u, v) ? (__double2hiint(h) & 0x7fffffff) : kInfHi;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {  // w = B_k - P; closest point B_k + t E_k
        const double wx = bt(F_V + 3 * k) - px, wy = bt(F_V + 3 * k + 1) - py, wz = bt(F_V + 3 * k + 2) - pz;
        const double ex = bt(F_E + 3 * k), ey = bt(F_E + 3 * k + 1), ez = bt(F_E + 3 * k + 2);
        const double t = clamp01(-fma(ex, wx, fma(ey, wy, ez * wz)) * bt(F_IL + k));
        const double dx = fma(t, ex, wx), dy = fma(t, ey, wy), dz = fma(t, ez, wz);
        best = min(best, __double2hiint(fma(dx, dx, fma(dy, dy, dz * dz))));
    }
    const double hv = __hiloint2double(hmin, 0);
    return min(best, __double2hiint(hv * hv));
}

// segment P0 + s D vs face B: both endpoints vs the face, the piercing test,
// and the three clamped segment/edge distances (Ericson, as in pair_d2).
template <class P>
__device__ __forceinline__ int seg_d2(const double p0[3], const double d[3], double Ld, double ILd, const P& bt) {
    int best = kInfHi, hmin = kInfHi;
    double w[3][3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        w[k][0] = bt(F_V + 3 * k) - p0[0];
        w[k][1] = bt(F_V + 3 * k + 1) - p0[1];
        w[k][2] = bt(F_V + 3 * k + 2) - p0[2];
    }
    {
        const double nb[3] = {bt(F_N), bt(F_N + 1), bt(F_N + 2)};
        const double ub[3] = {bt(F_U), bt(F_U + 1), bt(F_U + 2)};
        const double vb[3] = {bt(F_W), bt(F_W + 1), bt(F_W + 2)};
        // endpoint 0: P0 - B0 = -w0 ; endpoint 1: P1 - B0 = D - w0
        const double h0 = -dot3(nb, w[0][0], w[0][1], w[0][2]);
        const double u0 = -dot3(ub, w[0][0], w[0][1], w[0][2]);
        const double v0 = -dot3(vb, w[0][0], w[0][1], w[0][2]);
        const double h1 = h0 + dot3(nb, d[0], d[1], d[2]);
        const double u1 = u0 + dot3(ub, d[0], d[1], d[2]);
        const double v1 = v0 + dot3(vb, d[0], d[1], d[2]);
        hmin = min(inside(u0, v0) ? (__double2hiint(h0) & 0x7fffffff) : kInfHi,
                   inside(u1, v1) ? (__double2hiint(h1) & 0x7fffffff) : kInfHi);
        // piercing: X = P0 + l D with l = h0/(h0-h1); u(X)(h0-h1) = h0 u1 - h1 u0
        const double D = h0 - h1;
        if ((__double2hiint(h0) ^ __double2hiint(h1)) < 0 && D != 0.0) {
            const double uD = fma(h0, u1, -h1 * u0), vD = fma(h0, v1, -h1 * v0), tD = D - uD - vD;
            const bool hit = D > 0.0 ? (uD >= 0.0 && vD >= 0.0 && tD >= 0.0) : (uD <= 0.0 && vD <= 0.0 && tD <= 0.0);
            if (hit) best = 0;
        }
    }
    double cw = dot3(d, w[0][0], w[0][1], w[0][2]);
#pragma unroll
    for (int k = 0; k < 3; ++k) {  // edge B_k -> B_k+1 vs the segment
        const double ebx = bt(F_E + 3 * k), eby = bt(F_E + 3 * k + 1), ebz = bt(F_E + 3 * k + 2);
        const double ILb = bt(F_IL + k);
        const double fw = fma(ebx, w[k][0], fma(eby, w[k][1], ebz * w[k][2]));
        const double bb = dot3(d, ebx, eby, ebz);
        const double bbI = bb * ILb;
        const double den = fma(-bbI, bb, Ld);
        const double num = fma(-bbI, fw, cw);
        double s = clamp01_hi(num * rcp_approx(den));
        const double t = clamp01(fma(bb, s, -fw) * ILb);
        s = clamp01(fma(bb, t, cw) * ILd);
        const double dx = fma(s, d[0], fma(-t, ebx, -w[k][0]));
        const double dy = fma(s, d[1], fma(-t, eby, -w[k][1]));
        const double dz = fma(s, d[2], fma(-t, ebz, -w[k][2]));
        best = min(best, __double2hiint(fma(dx, dx, fma(dy, dy, dz * dz))));
        cw += bb;  // cw_{k+1} = D.(w_k + Eb_k)
    }
    const double hv = __hiloint2double(hmin, 0);
    return min(best, __double2hiint(hv * hv));
}

struct QueryRegs {
    double p0[3], d[3], Ld, ILd;
    bool point;  // a point query, or a zero-length segment (kernels.cpp:388)
};

__device__ __forceinline__ QueryRegs load_query(const QArgs& a, uint64_t q) {
    QueryRegs r;
#pragma unroll
    for (int k = 0; k < 3; ++k) r.p0[k] = __ldg(a.Q + (uint64_t)k * a.Qpad + q);
    if (a.kind == QK_SEG) {
        double p1[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) p1[k] = __ldg(a.Q + (uint64_t)(3 + k) * a.Qpad + q);
        r.point = p1[0] == r.p0[0] && p1[1] == r.p0[1] && p1[2] == r.p0[2];
#pragma unroll
        for (int k = 0; k < 3; ++k) r.d[k] = p1[k] - r.p0[k];
    } else {
        r.point = true;
        r.d[0] = r.d[1] = r.d[2] = 0.0;
    }
    r.Ld = fma(r.d[0], r.d[0], fma(r.d[1], r.d[1], r.d[2] * r.d[2]));
    r.ILd = r.Ld > 0.0 ? 1.0 / r.Ld : 0.0;
    return r;
}

template <class P>
__device__ __forceinline__ double query_d2(const QueryRegs& Q, const P& bt) {
    const int h = Q.point ? pt_d2(Q.p0[0], Q.p0[1], Q.p0[2], bt) : seg_d2(Q.p0, Q.d, Q.Ld, Q.ILd, bt);
    return __hiloint2double(h, 0);
}

__global__ void __launch_bounds__(kTile, 4) q_filter_kernel(QArgs a) {
    __shared__ alignas(128) double sm[2][NF * kSB];
    __shared__ alignas(8) uint64_t bar[2];
    __shared__ double red[kTile / 32];
    const uint64_t item = blockIdx.x;
    const uint64_t tl = item / a.n_chunks, ch = item - tl * a.n_chunks;
    const uint64_t q = min(tl * kTile + threadIdx.x, a.Qn - 1);
    const bool active = tl * kTile + threadIdx.x < a.Qn;
    const QueryRegs Q = load_query(a, q);
    const uint64_t b0 = ch * a.chunk, b1 = min(a.Bn, b0 + a.chunk);
    const int nsub = (int)((b1 - b0 + kSB - 1) / kSB);
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto issue = [&](int s) {
        const int st = s & 1;
        const uint64_t f0 = b0 + (uint64_t)s * kSB;
        const int cnt = (int)min((uint64_t)kSB, b1 - f0);
        const uint32_t bytes = (uint32_t)(((cnt + 1) & ~1) * sizeof(double));
        mbar_expect_tx(&bar[st], bytes * NF);
#pragma unroll 1
        for (int f = 0; f < NF; ++f) bulk_g2s(&sm[st][f * kSB], a.Bp + (uint64_t)f * a.Bn_pad + f0, bytes, &bar[st]);
    };
    if (threadIdx.x == 0) {
        issue(0);
        if (nsub > 1) issue(1);
    }
    double best = pos_inf();
#pragma unroll 1
    for (int s = 0; s < nsub; ++s) {
        const int st = s & 1;
        mbar_wait(&bar[st], (uint32_t)((s >> 1) & 1));
        const int cnt = (int)min((uint64_t)kSB, b1 - (b0 + (uint64_t)s * kSB));
        const double* sb = sm[st];
#pragma unroll 1
        for (int j = 0; j < cnt; ++j) {
            if (reinterpret_cast<const int*>(sb + F_DEG * kSB + j)[1] != 0) continue;  // degenerate face
            best = min_nn(best, query_d2(Q, FaceRef{sb + j, (uint64_t)kSB}));
        }
        __syncthreads();
        if (threadIdx.x == 0 && s + 2 < nsub) issue(s + 2);
    }
    if (!active) best = pos_inf();
    if (active && best < pos_inf()) atomicMin(a.qmin + q, (unsigned long long)__double_as_longlong(best));
    double m = best;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = min_nn(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double r = red[0];
#pragma unroll
        for (int w = 1; w < kTile / 32; ++w) r = min_nn(r, red[w]);
        a.itemmin[item] = r;
    }
}

// eta of one query: max edge over B and the segment, max |coord| over both
__device__ __forceinline__ double q_eta(const QArgs& a, uint64_t q, const double* Bs) {
    const QueryRegs Q = load_query(a, q);
    double ext = fmax(fabs(Q.p0[0]), fmax(fabs(Q.p0[1]), fabs(Q.p0[2])));
    ext = fmax(ext, fmax(fabs(Q.p0[0] + Q.d[0]), fmax(fabs(Q.p0[1] + Q.d[1]), fabs(Q.p0[2] + Q.d[2]))));
    return kBandEdge * fmax(Bs[6], sqrt(Q.Ld)) + kBandAbs * fmax(Bs[7], ext);
}

__global__ void q_band_kernel(QArgs a, const double* Bs, double* band2, double* band, unsigned long long* qD,
                              unsigned long long* qP) {
    const uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= a.Qn) return;
    qD[q] = kNone;
    qP[q] = kNone;
    const unsigned long long e = a.qmin[q];
    if (e == kNone) {
        band2[q] = band[q] = -1.0;
        return;
    }
    const double b = sqrt(__longlong_as_double((long long)e)) * (1.0 + kBandRel) + 2.0 * q_eta(a, q, Bs);
    band[q] = b;
    band2[q] = b * b * (1.0 + 4e-16);
}

__global__ void q_flag_kernel(QArgs a, uint64_t n_items, const double* band2, unsigned long long* list,
                              unsigned long long* count) {
    const uint64_t item = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (item >= n_items) return;
    const uint64_t tl = item / a.n_chunks;
    const uint64_t q0 = tl * kTile, q1 = min(a.Qn, q0 + kTile);
    double bmax = -1.0;
    for (uint64_t q = q0; q < q1; ++q) bmax = fmax(bmax, band2[q]);
    if (bmax >= 0.0 && a.itemmin[item] <= bmax) list[atomicAdd(count, 1ull)] = item;
}

__device__ __forceinline__ exact::tri tri_at(const double* P, uint64_t pad, uint64_t i) {
    double v[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) v[k] = __ldg(P + (uint64_t)(F_V + k) * pad + i);
    return exact::tri{{v[0], v[1], v[2]}, {v[3], v[4], v[5]}, {v[6], v[7], v[8]}};
}

__global__ void __launch_bounds__(kTile) q_verify_kernel(QArgs a, const unsigned long long* list,
                                                         const unsigned long long* count, int nsplit, int pass,
                                                         const double* band2, unsigned long long* qD,
                                                         unsigned long long* qP, unsigned long long* ncand) {
    const uint64_t units = *count * (uint64_t)nsplit;
    for (uint64_t w = blockIdx.x; w < units; w += gridDim.x) {
        const uint64_t item = list[w / nsplit];
        const int part = (int)(w % nsplit);
        const uint64_t tl = item / a.n_chunks, ch = item - tl * a.n_chunks;
        const uint64_t q = min(tl * kTile + threadIdx.x, a.Qn - 1);
        const bool active = tl * kTile + threadIdx.x < a.Qn;
        const QueryRegs Q = load_query(a, q);
        const uint64_t c0 = ch * a.chunk, c1 = min(a.Bn, c0 + a.chunk);
        const uint64_t len = (c1 - c0 + nsplit - 1) / nsplit;
        const uint64_t b0 = c0 + part * len, b1 = min(c1, b0 + len);
        const double b2 = active ? band2[q] : -1.0;
        const exact::v3 p0{Q.p0[0], Q.p0[1], Q.p0[2]};
        const exact::v3 p1{Q.p0[0] + Q.d[0], Q.p0[1] + Q.d[1], Q.p0[2] + Q.d[2]};
        for (uint64_t j = b0; j < b1; ++j) {
            if (__ldg(a.Bp + (uint64_t)F_DEG * a.Bn_pad + j) != 0.0) continue;
            const double d2 = query_d2(Q, FaceRefLdg{a.Bp + j, a.Bn_pad});
            if (d2 <= b2) {
                const exact::tri t = tri_at(a.Bp, a.Bn_pad, j);
                // the exact endpoints: p1 re-read (p0 + (p1 - p0) need not round-trip)
                exact::v3 e1 = p0;
                if (a.kind == QK_SEG)
                    e1 = exact::v3{__ldg(a.Q + 3 * a.Qpad + q), __ldg(a.Q + 4 * a.Qpad + q), __ldg(a.Q + 5 * a.Qpad + q)};
                const double dx = a.kind == QK_SEG ? exact::seg_tri(p0, e1, t).d : exact::pt_tri(p0, t).d;
                const unsigned long long bits = (unsigned long long)__double_as_longlong(dx);
                if (pass == 1) {
                    atomicMin(qD + q, bits);
                    atomicAdd(ncand, 1ull);
                } else if (bits == qD[q]) {
                    atomicMin(qP + q, (unsigned long long)j);
                }
            }
        }
        (void)p1;
    }
}

__global__ void q_check_kernel(QArgs a, const double* Bs, double* band2, double* band, unsigned long long* qD,
                               unsigned long long* qP, unsigned long long* retry) {
    const uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= a.Qn) return;
    const double b = band[q];
    if (b < 0.0) {
        band2[q] = -1.0;
        return;
    }
    const double eta = q_eta(a, q, Bs);
    const unsigned long long d = qD[q];
    if (d != kNone && __longlong_as_double((long long)d) > b - eta) {
        const double nb = __longlong_as_double((long long)d) * (1.0 + kBandRel) + 2.0 * eta;
        band[q] = nb;
        band2[q] = nb * nb * (1.0 + 4e-16);
        qD[q] = kNone;
        qP[q] = kNone;
        atomicAdd(retry, 1ull);
    } else {
        band2[q] = -1.0;
    }
}

// ---- intersects -------------------------------------------------------------
__global__ void __launch_bounds__(kTile, 4) q_hit_kernel(QArgs a, const double* Bs, unsigned long long* qhit,
                                                         unsigned long long* nexact) {
    __shared__ alignas(128) double sm[2][14 * kSB];
    __shared__ alignas(8) uint64_t bar[2];
    const int planes[14] = {0, 1, 2, 3, 4, 5, 6, 7, 8, F_N, F_N + 1, F_N + 2, F_C, F_DEG};
    const uint64_t item = blockIdx.x;
    const uint64_t tl = item / a.n_chunks, ch = item - tl * a.n_chunks;
    const uint64_t q = min(tl * kTile + threadIdx.x, a.Qn - 1);
    const uint64_t b0 = ch * a.chunk, b1 = min(a.Bn, b0 + a.chunk);
    double p0[3], p1[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        p0[k] = __ldg(a.Q + (uint64_t)k * a.Qpad + q);
        p1[k] = __ldg(a.Q + (uint64_t)(3 + k) * a.Qpad + q);
    }
    // cull margin over the bounding box of B and this segment (intersects.cu)
    double diag2 = 0.0, ext = Bs[7];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double lo = fmin(Bs[k], fmin(p0[k], p1[k])), hi = fmax(Bs[3 + k], fmax(p0[k], p1[k]));
        diag2 += (hi - lo) * (hi - lo);
        ext = fmax(ext, fmax(fabs(p0[k]), fabs(p1[k])));
    }
    const double tau = kCullDiag * sqrt(diag2) + kCullAbs * ext;
    bool live = tl * kTile + threadIdx.x < a.Qn && *(volatile unsigned long long*)(qhit + q) >= b0;
    if (!__syncthreads_or(live)) return;
    const int nsub = (int)((b1 - b0 + kSB - 1) / kSB);
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto issue = [&](int s) {
        const int st = s & 1;
        const uint64_t f0 = b0 + (uint64_t)s * kSB;
        const int cnt = (int)min((uint64_t)kSB, b1 - f0);
        const uint32_t bytes = (uint32_t)(((cnt + 1) & ~1) * sizeof(double));
        mbar_expect_tx(&bar[st], bytes * 14);
#pragma unroll 1
        for (int f = 0; f < 14; ++f)
            bulk_g2s(&sm[st][f * kSB], a.Bp + (uint64_t)planes[f] * a.Bn_pad + f0, bytes, &bar[st]);
    };
    if (threadIdx.x == 0) {
        issue(0);
        if (nsub > 1) issue(1);
    }
    unsigned long long nex = 0;
    const exact::v3 e0{p0[0], p0[1], p0[2]}, e1{p1[0], p1[1], p1[2]};
#pragma unroll 1
    for (int s = 0; s < nsub; ++s) {
        const int st = s & 1;
        mbar_wait(&bar[st], (uint32_t)((s >> 1) & 1));
        const uint64_t f0 = b0 + (uint64_t)s * kSB;
        const int cnt = (int)min((uint64_t)kSB, b1 - f0);
        const double* sb = sm[st];
        if (live && *(volatile unsigned long long*)(qhit + q) < f0) live = false;
        if (__syncthreads_or(live)) {
#pragma unroll 1
            for (int j = 0; j < cnt; ++j) {
                if (!live) continue;
                const double n0 = sb[9 * kSB + j], n1 = sb[10 * kSB + j], n2 = sb[11 * kSB + j], c = sb[12 * kSB + j];
                const double h0 = fma(n0, p0[0], fma(n1, p0[1], fma(n2, p0[2], -c)));
                const double h1 = fma(n0, p1[0], fma(n1, p1[1], fma(n2, p1[2], -c)));
                const double q0 = fabs(h0) - tau, q1 = fabs(h1) - tau;
                const bool apart = ((__double2hiint(h0) ^ __double2hiint(h1)) | __double2hiint(q0) |
                                    __double2hiint(q1)) >= 0 &&
                                   q0 != 0.0 && q1 != 0.0;
                // degenerate faces have n = 0, c = 0: never culled, decided exactly
                if (apart) continue;
                ++nex;
                const double* bv = sb + j;
                const exact::tri t{{bv[0], bv[kSB], bv[2 * kSB]}, {bv[3 * kSB], bv[4 * kSB], bv[5 * kSB]},
                                   {bv[6 * kSB], bv[7 * kSB], bv[8 * kSB]}};
                if (exact::seg_tri_hit(e0, e1, t)) {
                    atomicMin(qhit + q, (unsigned long long)(f0 + j));
                    live = false;  // later faces only give larger indices
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && s + 2 < nsub) issue(s + 2);
    }
    if (nex) atomicAdd(nexact, nex);
}

// queries (host AoS, width 6 or 3) -> SoA planes
__global__ void q_transpose_kernel(const double* __restrict__ in, uint64_t n, int width, uint64_t pad,
                                   double* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int k = 0; k < width; ++k) out[(uint64_t)k * pad + i] = in[(uint64_t)width * i + k];
}

}  // namespace

void run_queries(const Ctx& cx, int kind, int op, const double* host_q, uint64_t n, const Geom& B, double* dist,
                 uint8_t* hit, uint64_t* face) {
    const cudaStream_t st = cx.stream;
    tdb_stats& S = *cx.stats;
    std::memset(&S, 0, sizeof S);
    for (uint64_t q = 0; q < n; ++q) {
        if (dist) dist[q] = pos_inf_h();
        if (hit) hit[q] = 0;
        face[q] = kNone;
    }
    if (n == 0 || B.n == 0) return;
    const int width = kind == QK_SEG ? 6 : 3;
    const uint64_t pad = ((n + kPlanePad - 1) / kPlanePad) * kPlanePad;
    const uint64_t tiles = (n + kTile - 1) / kTile;
    const uint64_t chunk = pick_chunk(tiles, B.n, cx.sms, 16);
    const uint64_t n_chunks = (B.n + chunk - 1) / chunk;
    const uint64_t n_items = tiles * n_chunks;
    if (n_items > 0x7fffffffull) throw std::invalid_argument("queries: too many work items for one launch");

    double *stage = nullptr, *Q = nullptr, *Bs = nullptr;
    CK(cudaMallocAsync(&stage, n * width * sizeof(double), st));
    CK(cudaMallocAsync(&Q, pad * width * sizeof(double), st));
    CK(cudaMallocAsync(&Bs, kObjStats * sizeof(double), st));
    CK(cudaMemcpyAsync(stage, host_q, n * width * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(Bs, B.stats, kObjStats * sizeof(double), cudaMemcpyHostToDevice, st));
    cudaEvent_t ev[4];
    for (auto& e : ev) CK(cudaEventCreate(&e));
    CK(cudaEventRecord(ev[0], st));
    q_transpose_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(stage, n, width, pad, Q);
    CK(cudaGetLastError());
    QArgs a{Q, n, pad, kind, B.planes, B.n_pad, B.n, n_chunks, chunk, nullptr, nullptr};
    std::vector<unsigned long long> hres(n);
    uint64_t launches = 1, flagged = 0;
    int rounds = 0;
    unsigned long long hc[4] = {0, 0, 0, 0};
    std::vector<void*> mem = {stage, Q, Bs};
    auto alloc = [&](size_t bytes) {
        void* p = nullptr;
        CK(cudaMallocAsync(&p, std::max<size_t>(1, bytes), st));
        mem.push_back(p);
        return p;
    };
    unsigned long long* ctr = (unsigned long long*)alloc(4 * sizeof(unsigned long long));
    CK(cudaMemsetAsync(ctr, 0, 4 * sizeof(unsigned long long), st));
    if (op == TDB_OP_INTERSECTS) {
        unsigned long long* qhit = (unsigned long long*)alloc(n * sizeof(unsigned long long));
        CK(cudaMemsetAsync(qhit, 0xff, n * sizeof(unsigned long long), st));
        q_hit_kernel<<<(unsigned)n_items, kTile, 0, st>>>(a, Bs, qhit, ctr);
        CK(cudaGetLastError());
        CK(cudaEventRecord(ev[1], st));
        CK(cudaEventRecord(ev[2], st));
        CK(cudaMemcpyAsync(hres.data(), qhit, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(hc, ctr, sizeof hc, cudaMemcpyDeviceToHost, st));
        launches += 1;
        rounds = 1;
        S.exact_pairs = hc[0];
    } else {
        a.itemmin = (double*)alloc(n_items * sizeof(double));
        a.qmin = (unsigned long long*)alloc(n * sizeof(unsigned long long));
        double* band2 = (double*)alloc(n * sizeof(double));
        double* band = (double*)alloc(n * sizeof(double));
        unsigned long long* qD = (unsigned long long*)alloc(n * sizeof(unsigned long long));
        unsigned long long* qP = (unsigned long long*)alloc(n * sizeof(unsigned long long));
        unsigned long long* list = (unsigned long long*)alloc(n_items * sizeof(unsigned long long));
        CK(cudaMemsetAsync(a.qmin, 0xff, n * sizeof(unsigned long long), st));
        q_filter_kernel<<<(unsigned)n_items, kTile, 0, st>>>(a);
        CK(cudaGetLastError());
        CK(cudaEventRecord(ev[1], st));
        const unsigned qb = (unsigned)((n + 255) / 256);
        q_band_kernel<<<qb, 256, 0, st>>>(a, Bs, band2, band, qD, qP);
        CK(cudaGetLastError());
        launches += 2;
        for (;;) {
            ++rounds;
            CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st));
            CK(cudaMemsetAsync(ctr + 2, 0, sizeof(unsigned long long), st));
            q_flag_kernel<<<(unsigned)((n_items + 255) / 256), 256, 0, st>>>(a, n_items, band2, list, ctr);
            CK(cudaGetLastError());
            for (int pass = 1; pass <= 2; ++pass) {
                q_verify_kernel<<<(unsigned)(cx.sms * 8), kTile, 0, st>>>(a, list, ctr, 4, pass, band2, qD, qP,
                                                                          ctr + 1);
                CK(cudaGetLastError());
            }
            q_check_kernel<<<qb, 256, 0, st>>>(a, Bs, band2, band, qD, qP, ctr + 2);
            CK(cudaGetLastError());
            launches += 4;
            CK(cudaMemcpyAsync(hc, ctr, sizeof hc, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            flagged += hc[0];
            if (hc[2] == 0 || rounds >= 8) break;
        }
        CK(cudaEventRecord(ev[2], st));
        std::vector<unsigned long long> hd(n);
        CK(cudaMemcpyAsync(hd.data(), qD, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(hres.data(), qP, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (uint64_t q = 0; q < n; ++q)
            if (hres[q] != kNone) std::memcpy(&dist[q], &hd[q], sizeof(double));
        S.candidates = hc[1];
    }
    CK(cudaEventRecord(ev[3], st));
    for (void* p : mem) CK(cudaFreeAsync(p, st));
    CK(cudaStreamSynchronize(st));
    for (uint64_t q = 0; q < n; ++q) {
        face[q] = hres[q];
        if (hit) hit[q] = hres[q] != kNone;
    }
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, ev[0], ev[1]));
    S.ms_filter = ms;
    CK(cudaEventElapsedTime(&ms, ev[1], ev[2]));
    S.ms_verify = ms;
    CK(cudaEventElapsedTime(&ms, ev[0], ev[3]));
    S.ms_total = ms;
    for (auto& e : ev) cudaEventDestroy(e);
    S.pairs = n * B.n;
    S.pairs_evaluated = n * B.n;
    S.items = n_items;
    S.items_flagged = flagged;
    S.kernels = launches;
    S.rounds = rounds;
}

}  // namespace tdb
