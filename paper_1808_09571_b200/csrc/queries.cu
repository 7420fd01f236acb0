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
// Layout: a query set lives in HBM as SoA planes (uploaded once, reusable);
// a CTA holds 128 queries (one per thread) and streams the mesh through
// shared memory with TMA bulk copies. Filter values are high-word truncated
// squared distances (fast_pair.cuh conventions); the exact pass re-evaluates,
// with the bit-exact reference primitives (exact.cuh), every (query, face)
// whose filter value lies inside the query's band.
//
// Two distance paths:
//   * fused (the mesh fits one work chunk, e.g. the paper's 500-face ore):
//     one kernel — filter over the mesh, the query's band from its own
//     minimum, an exact rescan of the in-band faces, the band check — every
//     answer final inside the CTA;
//   * chunked (large meshes): filter -> per-query band -> flagged items ->
//     exact rescans (as distance.cu).
#include <algorithm>
#include <cstring>
#include <vector>

#include "exact.cuh"
#include "runtime.h"
#include "tma.cuh"

namespace tdb {

namespace {

constexpr unsigned long long kNone = ~0ull;
constexpr int kCand = 8;  // per-query candidate list of the fused kernel

struct QArgs {
    const double* Q;  // query planes: 6 (segments: p0 xyz, p1 xyz) or 3 (points), stride Qpad
    uint64_t Qn, Qpad;
    int kind;
    const double* Bp;
    uint64_t Bn_pad, Bn, n_chunks, chunk;
    double* itemmin;
    unsigned long long* qmin;
    // per B object: 1 = evaluate its degenerate faces (the reference's
    // TriangleMesh::has_degenerate_faces is false, kernels.cpp:350,357),
    // 0 = skip them
    const uint8_t* keep_deg;
};

// face j of the staged sub-tile is skipped: degenerate and its object skips them
__device__ __forceinline__ bool skip_face(const QArgs& a, const double* sb, int j, uint32_t obj = 0) {
    return reinterpret_cast<const int*>(sb + F_DEG * kSB + j)[1] != 0 && !a.keep_deg[obj];
}

// ---- TMA-staged streaming of B faces [b0, b1) through 2 SMEM stages ------
// `g` counts sub-tiles across calls so the mbarrier phases stay consistent
// when one kernel streams the same range several times.
template <int NP, int NS = 2>
struct Stream {
    // NS staged sub-tiles in flight. NS == 2: a CTA barrier per sub-tile.
    // NS > 2: each warp releases a stage through an "empty" mbarrier
    // (blockDim / 32 arrivals) and thread 0 refills the stage every warp
    // released NS - 2 sub-tiles earlier, so warps whose lanes meet exact
    // predicates may drift NS - 2 sub-tiles apart instead of meeting at a
    // barrier per sub-tile (one CTA barrier at the end of run()).
    double (*sm)[NP * kSB];
    uint64_t* bar;   // NS full barriers
    uint64_t* ebar;  // NS empty barriers (NS > 2)
    const int* plane;
    uint32_t g = 0;

    __device__ void init() {
        if (threadIdx.x == 0) {
#pragma unroll
            for (int i = 0; i < NS; ++i) {
                mbar_init(&bar[i], 1);
                if (NS > 2) mbar_init(&ebar[i], blockDim.x / 32);
            }
            mbar_fence_init();
        }
        __syncthreads();
    }

    __device__ void issue(const double* Bp, uint64_t pad, uint64_t b0, uint64_t b1, uint32_t s) {
        const int st = (g + s) % NS;
        const uint64_t f0 = b0 + (uint64_t)s * kSB;
        const int cnt = (int)min((uint64_t)kSB, b1 - f0);
        const uint32_t bytes = (uint32_t)(((cnt + 1) & ~1) * sizeof(double));
        mbar_expect_tx(&bar[st], bytes * NP);
#pragma unroll 1
        for (int f = 0; f < NP; ++f) bulk_g2s(&sm[st][f * kSB], Bp + (uint64_t)plane[f] * pad + f0, bytes, &bar[st]);
    }

    // fn(sb, cnt, f0) per staged sub-tile; must be called by every thread
    template <class F>
    __device__ void run(const double* Bp, uint64_t pad, uint64_t b0, uint64_t b1, F&& fn) {
        const uint32_t nsub = (uint32_t)((b1 - b0 + kSB - 1) / kSB);
        if (threadIdx.x == 0)
            for (uint32_t s = 0; s < min((uint32_t)NS, nsub); ++s) issue(Bp, pad, b0, b1, s);
#pragma unroll 1
        for (uint32_t s = 0; s < nsub; ++s) {
            const int st = (g + s) % NS;
            mbar_wait(&bar[st], ((g + s) / NS) & 1);
            const uint64_t f0 = b0 + (uint64_t)s * kSB;
            fn(sm[st], (int)min((uint64_t)kSB, b1 - f0), f0);
            if (NS == 2) {
                __syncthreads();
                if (threadIdx.x == 0 && s + 2 < nsub) issue(Bp, pad, b0, b1, s + 2);
            } else {
                __syncwarp();
                if ((threadIdx.x & 31) == 0) mbar_arrive(&ebar[st]);
                const int q = (int)s - (NS - 2);
                if (threadIdx.x == 0 && q >= 0 && (uint32_t)q + NS < nsub) {
                    mbar_wait(&ebar[(g + q) % NS], ((g + q) / NS) & 1);
                    issue(Bp, pad, b0, b1, q + NS);
                }
            }
        }
        if (NS > 2) __syncthreads();  // every stage released before a later run() refills it
        g += nsub;
    }
};

__device__ __constant__ int kDistPlaneIds[kFilterPlanes] = {0,  1,  2,  3,  4,  5,  6,  7,  8,  9,  10, 11,
                                                             12, 13, 14, 15, 16, 17, 18, 19, 20, 21, 22, 23,
                                                             24, 25, 26, 27, 28, 29, 30, 31, 32, 33, 34};
constexpr int kHitPlanes = 21;  // V (9), N (3), C, DEG, face AABB lo/hi (6), K
__device__ __constant__ int kHitPlaneIds[kHitPlanes] = {0,    1,        2,        3,    4,        5,        6,
                                                         7,    8,        F_N,      F_N + 1, F_N + 2, F_C,   F_DEG,
                                                         F_LO, F_LO + 1, F_LO + 2, F_HI, F_HI + 1, F_HI + 2, F_K};
enum { HP_N = 9, HP_C = 12, HP_DEG = 13, HP_LO = 14, HP_HI = 17, HP_K = 20 };

// Segment x face intersects cull: the pair's box diagonal D
// (segment box u face box) bounds every length in the reference's solve; the
// reference cannot hit when (1) the boxes are apart by kApart D, or (2) both
// endpoints lie beyond (kCullTwo + kappa) D on one side of the face plane
// (its t-test fails despite its own rounding). slo/shi: the segment's box.
__device__ __forceinline__ bool seg_face_culled(const double* p0, const double* p1, const double* slo,
                                                const double* shi, const double flo[3], const double fhi[3],
                                                double n0, double n1, double n2, double c, double kappa,
                                                double abs_tol) {
    double d2 = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double e = fmax(shi[k], fhi[k]) - fmin(slo[k], flo[k]);
        d2 = fma(e, e, d2);
    }
    const double D = sqrt(d2) * (1.0 + 1e-15);
    const double gap = kApart * D + abs_tol;
    bool apart = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) apart |= (flo[k] > shi[k] + gap) | (fhi[k] < slo[k] - gap);
    if (apart) return true;
    const double tau = (kCullTwo + kappa) * D + abs_tol;
    const double h0 = fma(n0, p0[0], fma(n1, p0[1], fma(n2, p0[2], -c)));
    const double h1 = fma(n0, p1[0], fma(n1, p1[1], fma(n2, p1[2], -c)));
    return (h0 > tau && h1 > tau) || (h0 < -tau && h1 < -tau);
}

// ---- filter values -----------------------------------------------------------
// point P vs face B: vertex/face projection + the three clamped point/edge
// distances.
template <class P>
__device__ __forceinline__ int pt_d2(double px, double py, double pz, const P& bt) {
    const double qx = px - bt(F_V), qy = py - bt(F_V + 1), qz = pz - bt(F_V + 2);
    int best = kInfHi, hmin;
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
    int best = kInfHi, hmin;
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
        double s = clamp01(num * rcp_nr(den));
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
    double p0[3], p1[3], d[3], Ld, ILd;
    bool point;  // a point query, or a zero-length segment (kernels.cpp:388)
};

__device__ __forceinline__ QueryRegs load_query(const QArgs& a, uint64_t q) {
    QueryRegs r;
#pragma unroll
    for (int k = 0; k < 3; ++k) r.p0[k] = __ldg(a.Q + (uint64_t)k * a.Qpad + q);
    if (a.kind == kQuerySegments) {
#pragma unroll
        for (int k = 0; k < 3; ++k) r.p1[k] = __ldg(a.Q + (uint64_t)(3 + k) * a.Qpad + q);
        r.point = r.p1[0] == r.p0[0] && r.p1[1] == r.p0[1] && r.p1[2] == r.p0[2];
    } else {
#pragma unroll
        for (int k = 0; k < 3; ++k) r.p1[k] = r.p0[k];
        r.point = true;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) r.d[k] = r.p1[k] - r.p0[k];
    r.Ld = fma(r.d[0], r.d[0], fma(r.d[1], r.d[1], r.d[2] * r.d[2]));
    r.ILd = r.Ld > 0.0 ? 1.0 / r.Ld : 0.0;
    return r;
}

template <class P>
__device__ __forceinline__ double query_d2(const QueryRegs& Q, const P& bt) {
    const int h = Q.point ? pt_d2(Q.p0[0], Q.p0[1], Q.p0[2], bt) : seg_d2(Q.p0, Q.d, Q.Ld, Q.ILd, bt);
    return __hiloint2double(h, 0);
}

// the reference primitive for one (query, face): distance bits
__device__ __forceinline__ unsigned long long exact_bits(const QueryRegs& Q, const double* sb, int j) {
    const double* bv = sb + j;
    const exact::tri t{{bv[0], bv[kSB], bv[2 * kSB]}, {bv[3 * kSB], bv[4 * kSB], bv[5 * kSB]},
                       {bv[6 * kSB], bv[7 * kSB], bv[8 * kSB]}};
    const exact::v3 p0{Q.p0[0], Q.p0[1], Q.p0[2]}, p1{Q.p1[0], Q.p1[1], Q.p1[2]};
    const double d = Q.point ? exact::pt_tri(p0, t).d : exact::seg_tri(p0, p1, t).d;
    return (unsigned long long)__double_as_longlong(d);
}

// eta(m) of one query (tdb_internal.h): max edge over B and the segment,
// B's max kappa, max |coord| over both. A band is complete when the exact
// minimum D has D + eta(D) <= band (distance.cu check_kernel).
__device__ __forceinline__ double q_eta(const QueryRegs& Q, const double* Bs, double m) {
    double ext = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) ext = fmax(ext, fmax(fabs(Q.p0[k]), fabs(Q.p1[k])));
    return band_eta_of(fmax(Bs[6], sqrt(Q.Ld)), Bs[8], fmax(Bs[7], ext), m);
}

// ---- fused path: the whole mesh is one chunk --------------------------------
#ifndef TDB_QF_MINB
#define TDB_QF_MINB 4  // 128 registers: 31.9 vs 34.9 ms at 3 on the paper workload (scripts/variants_q.sh)
#endif
__global__ void __launch_bounds__(kTile, TDB_QF_MINB) q_fused_kernel(QArgs a, const double* Bs, double* out_d,
                                                           unsigned long long* out_f, unsigned long long* ncand,
                                                           unsigned long long* nrounds, NearLog near) {
    __shared__ alignas(128) double sm[2][kFilterPlanes * kSB];
    __shared__ alignas(8) uint64_t bar[2];
    Stream<kFilterPlanes> S{sm, bar, nullptr, kDistPlaneIds};
    S.init();
    // per-thread candidate list (SMEM, column per thread): faces whose filter
    // value lies inside the band of the running minimum
    __shared__ double cd[kCand][kTile];
    __shared__ uint32_t cj[kCand][kTile];
    const int tx = threadIdx.x;
    const uint64_t qi = (uint64_t)blockIdx.x * kTile + tx;
    const bool active = qi < a.Qn;
    const uint64_t q = min(qi, a.Qn - 1);
    const QueryRegs Q = load_query(a, q);
    auto band_of = [&](double m2) {
        const double m = sqrt(m2);
        return m * (1.0 + kBandRel) + 2.0 * q_eta(Q, Bs, m);
    };
    auto widen = [&](double D) { return D * (1.0 + kBandRel) + 2.0 * q_eta(Q, Bs, D); };
    double best = pos_inf(), cut2 = pos_inf(), evicted = pos_inf();
    int nc = 0;
    S.run(a.Bp, a.Bn_pad, 0, a.Bn, [&](const double* sb, int cnt, uint64_t f0) {
        auto take = [&](double d2, int j) {  // candidate-list update for face f0 + j
            if (d2 < best) {  // new minimum: tighten the cut, drop what fell out of it
                best = d2;
                const double b = band_of(best);
                cut2 = b * b * (1.0 + 4e-16);
                int w = 0;
                for (int k = 0; k < nc; ++k)
                    if (cd[k][tx] <= cut2) cd[w][tx] = cd[k][tx], cj[w][tx] = cj[k][tx], ++w;
                nc = w;
            }
            if (d2 <= cut2) {
                if (nc < kCand) {
                    cd[nc][tx] = d2, cj[nc][tx] = (uint32_t)(f0 + j), ++nc;
                } else {  // full: keep the kCand smallest, remember the best one dropped
                    int worst = 0;
                    for (int k = 1; k < kCand; ++k)
                        if (cd[k][tx] > cd[worst][tx]) worst = k;
                    if (d2 < cd[worst][tx]) {
                        evicted = fmin(evicted, cd[worst][tx]);
                        cd[worst][tx] = d2, cj[worst][tx] = (uint32_t)(f0 + j);
                    } else {
                        evicted = fmin(evicted, d2);
                    }
                }
            }
        };
#pragma unroll 1
        for (int j = 0; j < cnt; ++j)
            if (!skip_face(a, sb, j)) take(query_d2(Q, FaceRef{sb + j, (uint64_t)kSB}), j);  // uniform
    });
    double band = active && best < pos_inf() ? band_of(best) : -1.0;
    unsigned long long D = kNone, P = kNone, cand = 0;
    bool again = false;
    if (band >= 0.0) {  // exact composition on the listed candidates, lanes in lockstep
        const double b2 = band * band * (1.0 + 4e-16);
        for (int k = 0; k < nc; ++k) {
            if (cd[k][tx] > b2) continue;
            ++cand;
            const uint64_t j = cj[k][tx];
            const exact::tri t = [&] {
                double v[9];
#pragma unroll
                for (int c = 0; c < 9; ++c) v[c] = __ldg(a.Bp + (uint64_t)(F_V + c) * a.Bn_pad + j);
                return exact::tri{{v[0], v[1], v[2]}, {v[3], v[4], v[5]}, {v[6], v[7], v[8]}};
            }();
            const exact::v3 p0{Q.p0[0], Q.p0[1], Q.p0[2]}, p1{Q.p1[0], Q.p1[1], Q.p1[2]};
            const double dx = Q.point ? exact::pt_tri(p0, t).d : exact::seg_tri(p0, p1, t).d;
            const unsigned long long e = (unsigned long long)__double_as_longlong(dx);
            if (e < D || (e == D && j < P)) D = e, P = j;
            if (Q.point ? exact::near_area(t) : exact::near_degenerate_seg(p0, p1, t)) near_log(near, q, j);
        }
        // complete only if nothing in the band was dropped and the band holds
        const double Dd = D != kNone ? __longlong_as_double((long long)D) : 0.0;
        const bool out = D != kNone && Dd + q_eta(Q, Bs, Dd) > band;
        again = evicted <= b2 || D == kNone || out;
        if (out) band = widen(Dd);
    }
    int rounds = 1;
    while (__syncthreads_or(again)) {  // fallback exact rescan (list overflow or a widened band)
        ++rounds;
        const double b2 = again ? band * band * (1.0 + 4e-16) : -1.0;
        if (again) D = P = kNone;
        S.run(a.Bp, a.Bn_pad, 0, a.Bn, [&](const double* sb, int cnt, uint64_t f0) {
#pragma unroll 1
            for (int j = 0; j < cnt; ++j) {
                if (skip_face(a, sb, j)) continue;
                if (b2 < 0.0) continue;
                if (query_d2(Q, FaceRef{sb + j, (uint64_t)kSB}) > b2) continue;
                ++cand;
                const unsigned long long e = exact_bits(Q, sb, j);
                if (e < D) D = e, P = f0 + j;  // ascending faces: strict < keeps the lowest index
            }
        });
        if (again) {
            const double Dd = D != kNone ? __longlong_as_double((long long)D) : 0.0;
            if (D != kNone && Dd + q_eta(Q, Bs, Dd) > band) {
                band = widen(Dd);
            } else {
                again = false;
            }
        }
        if (rounds >= 8) break;
    }
    if (active) {
        out_d[q] = P == kNone ? pos_inf() : __longlong_as_double((long long)D);
        out_f[q] = P;
    }
    if (cand) atomicAdd(ncand, cand);
    if (threadIdx.x == 0) atomicMax(nrounds, (unsigned long long)rounds);
}

// ---- chunked path -------------------------------------------------------------
__global__ void __launch_bounds__(kTile, 4) q_filter_kernel(QArgs a) {
    __shared__ alignas(128) double sm[2][kFilterPlanes * kSB];
    __shared__ alignas(8) uint64_t bar[2];
    __shared__ double red[kTile / 32];
    Stream<kFilterPlanes> S{sm, bar, nullptr, kDistPlaneIds};
    S.init();
    const uint64_t item = blockIdx.x;
    const uint64_t tl = item / a.n_chunks, ch = item - tl * a.n_chunks;
    const uint64_t q = min(tl * kTile + threadIdx.x, a.Qn - 1);
    const bool active = tl * kTile + threadIdx.x < a.Qn;
    const QueryRegs Q = load_query(a, q);
    const uint64_t b0 = ch * a.chunk, b1 = min(a.Bn, b0 + a.chunk);
    double best = pos_inf();
    S.run(a.Bp, a.Bn_pad, b0, b1, [&](const double* sb, int cnt, uint64_t) {
#pragma unroll 1
        for (int j = 0; j < cnt; ++j) {
            if (skip_face(a, sb, j)) continue;
            best = min_nn(best, query_d2(Q, FaceRef{sb + j, (uint64_t)kSB}));
        }
    });
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
    const double m = sqrt(__longlong_as_double((long long)e));
    const double b = m * (1.0 + kBandRel) + 2.0 * q_eta(load_query(a, q), Bs, m);
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

// exact rescan of flagged items, TMA-staged like the filter
template <class SS>
__device__ __forceinline__ void q_verify_item(const QArgs& a, SS& S, uint64_t item, int pass, const double* band2,
                                              unsigned long long* qD, unsigned long long* qP,
                                              unsigned long long* ncand, const NearLog& near) {
    const uint64_t tl = item / a.n_chunks, ch = item - tl * a.n_chunks;
    const uint64_t q = min(tl * kTile + threadIdx.x, a.Qn - 1);
    const bool active = tl * kTile + threadIdx.x < a.Qn;
    const QueryRegs Q = load_query(a, q);
    const uint64_t b0 = ch * a.chunk, b1 = min(a.Bn, b0 + a.chunk);
    const double b2 = active ? band2[q] : -1.0;
    unsigned long long cand = 0;
    S.run(a.Bp, a.Bn_pad, b0, b1, [&](const double* sb, int cnt, uint64_t f0) {
#pragma unroll 1
        for (int j = 0; j < cnt; ++j) {
            if (skip_face(a, sb, j)) continue;
            if (b2 < 0.0 || query_d2(Q, FaceRef{sb + j, (uint64_t)kSB}) > b2) continue;
            const unsigned long long e = exact_bits(Q, sb, j);
            if (pass == 1) {
                atomicMin(qD + q, e);
                ++cand;
                const double* bv = sb + j;
                const exact::tri t{{bv[0], bv[kSB], bv[2 * kSB]}, {bv[3 * kSB], bv[4 * kSB], bv[5 * kSB]},
                                   {bv[6 * kSB], bv[7 * kSB], bv[8 * kSB]}};
                const exact::v3 p0{Q.p0[0], Q.p0[1], Q.p0[2]}, p1{Q.p1[0], Q.p1[1], Q.p1[2]};
                if (Q.point ? exact::near_area(t) : exact::near_degenerate_seg(p0, p1, t)) near_log(near, q, f0 + j);
            } else if (e == qD[q]) {
                atomicMin(qP + q, (unsigned long long)(f0 + j));
            }
        }
    });
    if (cand) atomicAdd(ncand, cand);
}

// Grid-stride over the flagged items (the count stays on the device: no
// host round trip between the flag and verify passes).
__global__ void __launch_bounds__(kTile, 4) q_verify_kernel(QArgs a, const unsigned long long* list,
                                                            const unsigned long long* count, int pass,
                                                            const double* band2, unsigned long long* qD,
                                                            unsigned long long* qP, unsigned long long* ncand,
                                                            NearLog near) {
    __shared__ alignas(128) double sm[2][kFilterPlanes * kSB];
    __shared__ alignas(8) uint64_t bar[2];
    Stream<kFilterPlanes> S{sm, bar, nullptr, kDistPlaneIds};
    S.init();
    const uint64_t nflag = *count;
    for (uint64_t w = blockIdx.x; w < nflag; w += gridDim.x) q_verify_item(a, S, list[w], pass, band2, qD, qP, ncand, near);
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
    const QueryRegs Q = load_query(a, q);
    const unsigned long long d = qD[q];
    const double m = d != kNone ? __longlong_as_double((long long)d) : 0.0;
    if (d != kNone && m + q_eta(Q, Bs, m) > b) {
        const double nb = m * (1.0 + kBandRel) + 2.0 * q_eta(Q, Bs, m);
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
// Per (segment, face): (1) the segment's box vs the face's AABB plane,
// expanded by tau; (2) both endpoints strictly on one side of the face plane
// by tau; otherwise (3) the exact reference predicate. (1) and (2) only drop
// pairs the reference cannot hit (intersects.cu header); degenerate faces
// (n = 0, c = 0) always reach (3).
// sub-tiles in flight (Stream): the lanes that reach the exact predicate
// differ from warp to warp, so warps drift instead of meeting per sub-tile
#ifndef TDB_QHIT_STAGES
#define TDB_QHIT_STAGES 8
#endif
constexpr int kQHitStages = TDB_QHIT_STAGES;
__global__ void __launch_bounds__(kTile, 4) q_hit_kernel(QArgs a, const double* Bs, unsigned long long* qhit,
                                                         unsigned long long* nexact, NearLog near) {
    __shared__ alignas(128) double sm[kQHitStages][kHitPlanes * kSB];
    __shared__ alignas(8) uint64_t bar[kQHitStages], ebar[kQHitStages];
    Stream<kHitPlanes, kQHitStages> S{sm, bar, ebar, kHitPlaneIds};
    S.init();
    const uint64_t item = blockIdx.x;
    const uint64_t tl = item / a.n_chunks, ch = item - tl * a.n_chunks;
    const uint64_t q = min(tl * kTile + threadIdx.x, a.Qn - 1);
    const uint64_t b0 = ch * a.chunk, b1 = min(a.Bn, b0 + a.chunk);
    double p0[3], p1[3], lo[3], hi[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        p0[k] = __ldg(a.Q + (uint64_t)k * a.Qpad + q);
        p1[k] = __ldg(a.Q + (uint64_t)(3 + k) * a.Qpad + q);
    }
    double diag2 = 0.0, ext = Bs[7];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double l = fmin(Bs[k], fmin(p0[k], p1[k])), h = fmax(Bs[3 + k], fmax(p0[k], p1[k]));
        diag2 += (h - l) * (h - l);
        ext = fmax(ext, fmax(fabs(p0[k]), fabs(p1[k])));
        lo[k] = fmin(p0[k], p1[k]);
        hi[k] = fmax(p0[k], p1[k]);
    }
    // coarse box test against the whole mesh's diagonal (>= every pair's D)
    const double abs_tol = kCullAbs * ext, gap_mesh = kApart * sqrt(diag2) * (1.0 + 1e-15) + abs_tol;
    bool live = tl * kTile + threadIdx.x < a.Qn && *(volatile unsigned long long*)(qhit + q) >= b0;
    if (!__syncthreads_or(live)) return;
    unsigned long long nex = 0;
    const exact::v3 e0{p0[0], p0[1], p0[2]}, e1{p1[0], p1[1], p1[2]};
    S.run(a.Bp, a.Bn_pad, b0, b1, [&](const double* sb, int cnt, uint64_t f0) {
        if (live && *(volatile unsigned long long*)(qhit + q) < f0) live = false;
#pragma unroll 1
        for (int j = 0; j < cnt; ++j) {
            if (!live) continue;
            bool apart = false;
            double flo[3], fhi[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                flo[k] = sb[(HP_LO + k) * kSB + j], fhi[k] = sb[(HP_HI + k) * kSB + j];
                apart |= (flo[k] > hi[k] + gap_mesh) | (fhi[k] < lo[k] - gap_mesh);
            }
            if (apart) continue;
            if (seg_face_culled(p0, p1, lo, hi, flo, fhi, sb[HP_N * kSB + j], sb[(HP_N + 1) * kSB + j],
                                sb[(HP_N + 2) * kSB + j], sb[HP_C * kSB + j], sb[HP_K * kSB + j], abs_tol))
                continue;
            ++nex;
            const double* bv = sb + j;
            const exact::tri t{{bv[0], bv[kSB], bv[2 * kSB]}, {bv[3 * kSB], bv[4 * kSB], bv[5 * kSB]},
                               {bv[6 * kSB], bv[7 * kSB], bv[8 * kSB]}};
            if (exact::near_degenerate_seg(e0, e1, t)) near_log(near, q, f0 + j);
            if (exact::seg_tri_hit(e0, e1, t)) {
                atomicMin(qhit + q, (unsigned long long)(f0 + j));
                live = false;  // later faces only give larger indices
            }
        }
    });
    if (nex) atomicAdd(nexact, nex);
}

// final per-query outputs: distance (+inf when no face qualified) and hit
__global__ void q_finalize_kernel(uint64_t n, const unsigned long long* __restrict__ rD,
                                  const unsigned long long* __restrict__ rP, double* __restrict__ dist,
                                  uint8_t* __restrict__ hit) {
    const uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const bool found = rP[q] != kNone;
    if (dist) dist[q] = found && rD ? __longlong_as_double((long long)rD[q]) : pos_inf();
    if (hit) hit[q] = found ? 1 : 0;
}

// queries (host AoS, width 6 or 3) -> SoA planes
__global__ void q_transpose_kernel(const double* __restrict__ in, uint64_t n, int width, uint64_t pad,
                                   double* __restrict__ out, unsigned long long* __restrict__ nonfinite) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    bool bad = false;
    for (int k = 0; k < width; ++k) {
        const double x = in[(uint64_t)width * i + k];
        bad |= !isfinite(x);
        out[(uint64_t)k * pad + i] = x;
    }
    if (bad) atomicAdd(nonfinite, 1ull);
}

}  // namespace

void queries_build(QuerySet* qs, const double* host_q, uint64_t n, int kind, cudaStream_t st) {
    qs->n = n;
    qs->kind = kind;
    qs->width = kind == kQuerySegments ? 6 : 3;
    qs->pad = ((n + kPlanePad - 1) / kPlanePad) * kPlanePad;
    CK(cudaMallocAsync(&qs->planes, std::max<uint64_t>(1, qs->pad * qs->width) * sizeof(double), st));
    unsigned long long bad = 0;
    if (n) {
        double* stage = nullptr;
        unsigned long long* nbad = nullptr;
        CK(cudaMallocAsync(&stage, n * qs->width * sizeof(double), st));
        CK(cudaMallocAsync(&nbad, sizeof(unsigned long long), st));
        CK(cudaMemsetAsync(nbad, 0, sizeof(unsigned long long), st));
        h2d(stage, host_q, n * qs->width * sizeof(double), st);
        q_transpose_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(stage, n, qs->width, qs->pad, qs->planes,
                                                                       nbad);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&bad, nbad, sizeof bad, cudaMemcpyDeviceToHost, st));
        CK(cudaFreeAsync(stage, st));
        CK(cudaFreeAsync(nbad, st));
    }
    CK(cudaStreamSynchronize(st));
    if (bad)
        throw std::invalid_argument(std::to_string(bad) +
                                    " quer(ies) with non-finite coordinates (geometry.hpp:16-18 requires finite)");
}

void run_queries(const Ctx& cx, int op, const QuerySet& qs, const Geom& B, double* dist, uint8_t* hit,
                 uint64_t* face) {
    const cudaStream_t st = cx.stream;
    tdb_stats& S = *cx.stats;
    std::memset(&S, 0, sizeof S);
    const uint64_t n = qs.n;
    if (n == 0) return;
    if (B.n == 0) {
        for (uint64_t q = 0; q < n; ++q) {
            if (dist) dist[q] = pos_inf_h();
            if (hit) hit[q] = 0;
            face[q] = kNone;
        }
        return;
    }
    const uint64_t tiles = (n + kTile - 1) / kTile;
    const bool fused = op == TDB_OP_DISTANCE && B.n <= kChunk && tiles >= (uint64_t)cx.sms * 2;
    const uint64_t chunk = fused ? kChunk : pick_chunk(tiles, B.n, cx.sms, 16);
    const uint64_t n_chunks = (B.n + chunk - 1) / chunk;
    const uint64_t n_items = tiles * n_chunks;
    if (n_items > 0x7fffffffull) throw std::invalid_argument("queries: too many work items for one launch");

    std::vector<void*> mem;
    auto alloc = [&](size_t bytes) {
        void* p = nullptr;
        CK(cudaMallocAsync(&p, std::max<size_t>(1, bytes), st));
        mem.push_back(p);
        return p;
    };
    double* Bs = (double*)alloc(kObjStats * sizeof(double));
    CK(cudaMemcpyAsync(Bs, B.stats, kObjStats * sizeof(double), cudaMemcpyHostToDevice, st));
    unsigned long long* ctr = (unsigned long long*)alloc(4 * sizeof(unsigned long long));
    CK(cudaMemsetAsync(ctr, 0, 4 * sizeof(unsigned long long), st));
    // results: exact distance bits / face (or lowest hit face), finalized on the device
    unsigned long long* rD = (unsigned long long*)alloc(n * sizeof(unsigned long long));
    unsigned long long* rP = (unsigned long long*)alloc(n * sizeof(unsigned long long));
    NearDev near;
    near.alloc(st);
    cudaEvent_t* ev = thread_events().e;
    CK(cudaEventRecord(ev[0], st));
    QArgs a{qs.planes, n, qs.pad, qs.kind, B.planes, B.n_pad, B.n, n_chunks, chunk, nullptr, nullptr, B.d_keep_deg};
    uint64_t launches = 0, flagged = 0;
    int rounds = 0;
    unsigned long long hc[4] = {0, 0, 0, 0};
    if (op == TDB_OP_INTERSECTS) {
        CK(cudaMemsetAsync(rP, 0xff, n * sizeof(unsigned long long), st));
        q_hit_kernel<<<(unsigned)n_items, kTile, 0, st>>>(a, Bs, rP, ctr, near.log);
        CK(cudaGetLastError());
        CK(cudaEventRecord(ev[1], st));
        CK(cudaEventRecord(ev[2], st));
        launches = 1;
        rounds = 1;
    } else if (fused) {
        q_fused_kernel<<<(unsigned)tiles, kTile, 0, st>>>(a, Bs, (double*)rD, rP, ctr, ctr + 1, near.log);
        CK(cudaGetLastError());
        CK(cudaEventRecord(ev[1], st));
        CK(cudaEventRecord(ev[2], st));
        launches = 1;
    } else {
        a.itemmin = (double*)alloc(n_items * sizeof(double));
        a.qmin = (unsigned long long*)alloc(n * sizeof(unsigned long long));
        double* band2 = (double*)alloc(n * sizeof(double));
        double* band = (double*)alloc(n * sizeof(double));
        unsigned long long* list = (unsigned long long*)alloc(n_items * sizeof(unsigned long long));
        CK(cudaMemsetAsync(a.qmin, 0xff, n * sizeof(unsigned long long), st));
        q_filter_kernel<<<(unsigned)n_items, kTile, 0, st>>>(a);
        CK(cudaGetLastError());
        CK(cudaEventRecord(ev[1], st));
        const unsigned qb = (unsigned)((n + 255) / 256);
        q_band_kernel<<<qb, 256, 0, st>>>(a, Bs, band2, band, rD, rP);
        CK(cudaGetLastError());
        launches = 2;
        for (;;) {
            ++rounds;
            CK(cudaMemsetAsync(ctr + 2, 0, 2 * sizeof(unsigned long long), st));  // flagged, retry
            q_flag_kernel<<<(unsigned)((n_items + 255) / 256), 256, 0, st>>>(a, n_items, band2, list, ctr + 2);
            CK(cudaGetLastError());
            const unsigned vgrid = (unsigned)std::min<uint64_t>(n_items, (uint64_t)cx.sms * 4);
            for (int pass = 1; pass <= 2; ++pass) {
                q_verify_kernel<<<vgrid, kTile, 0, st>>>(a, list, ctr + 2, pass, band2, rD, rP, ctr, near.log);
                CK(cudaGetLastError());
            }
            q_check_kernel<<<qb, 256, 0, st>>>(a, Bs, band2, band, rD, rP, ctr + 3);
            CK(cudaGetLastError());
            launches += 4;
            CK(cudaMemcpyAsync(hc, ctr, sizeof hc, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            flagged += hc[2];
            if (hc[3] == 0 || rounds >= 8) break;
        }
        CK(cudaEventRecord(ev[2], st));
    }
    // distances as doubles (+inf when no face qualified), hits as bytes
    double* od = dist ? (double*)alloc(n * sizeof(double)) : nullptr;
    uint8_t* oh = hit ? (uint8_t*)alloc(n) : nullptr;
    q_finalize_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, op == TDB_OP_DISTANCE ? rD : nullptr, rP, od,
                                                                  oh);
    CK(cudaGetLastError());
    ++launches;
    CK(cudaEventRecord(ev[3], st));
    if (od) d2h(dist, od, n * sizeof(double), st);
    if (oh) d2h(hit, oh, n, st);
    d2h(face, rP, n * sizeof(uint64_t), st);
    CK(cudaMemcpyAsync(hc, ctr, sizeof hc, cudaMemcpyDeviceToHost, st));
    for (void* p : mem) CK(cudaFreeAsync(p, st));
    CK(cudaStreamSynchronize(st));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, ev[0], ev[1]));
    S.ms_filter = ms;
    CK(cudaEventElapsedTime(&ms, ev[1], ev[2]));
    S.ms_verify = ms;
    CK(cudaEventElapsedTime(&ms, ev[0], ev[3]));
    S.ms_total = ms;
    S.pairs = n * B.n;
    S.pairs_evaluated = n * B.n;
    S.items = n_items;
    S.items_flagged = flagged;
    if (op == TDB_OP_DISTANCE) S.candidates = hc[0];
    else S.exact_pairs = hc[0];
    S.kernels = launches;
    S.rounds = fused ? (int)hc[1] : rounds;
    near.fetch(st, cx.near);
    S.near_degenerate = cx.near->count;
}

// ---- one literal against every object of a table ----------------------------
// run_batch over Mesh records with a Segment / Point literal (batch.cpp:44-48,
// :59): per record, distance_to_mesh(literal, record mesh) (lowest face on
// ties, degenerate faces skipped, kernels.cpp:340-405) or intersects_mesh
// (lowest hit face, kernels.cpp:407-432). One CTA per 128-face tile of the
// table (tiles never straddle objects); the same filter -> band -> exact
// re-evaluation as the query sets, with per-object bands and the object's
// own AABB / scale header.
namespace {

// face f of object obj is skipped: degenerate and the object skips them
__device__ __forceinline__ bool face_skipped(const QArgs& a, const double* P, uint64_t pad, uint64_t f, uint32_t obj) {
    return reinterpret_cast<const int*>(P + (uint64_t)F_DEG * pad + f)[1] != 0 && !a.keep_deg[obj];
}

__device__ __forceinline__ exact::tri face_tri(const double* P, uint64_t pad, uint64_t f) {
    double v[9];
#pragma unroll
    for (int c = 0; c < 9; ++c) v[c] = __ldg(P + (uint64_t)(F_V + c) * pad + f);
    return exact::tri{{v[0], v[1], v[2]}, {v[3], v[4], v[5]}, {v[6], v[7], v[8]}};
}

__global__ void __launch_bounds__(kTile) lt_filter_kernel(QArgs a, const Tile* tiles, const double* P, uint64_t pad,
                                                          unsigned long long* objmin) {
    __shared__ double red[kTile / 32];
    const Tile T = tiles[blockIdx.x];
    const QueryRegs Q = load_query(a, 0);
    double d2 = pos_inf();
    if (threadIdx.x < T.count) {
        const uint64_t f = T.row0 + threadIdx.x;
        if (!face_skipped(a, P, pad, f, T.obj)) d2 = query_d2(Q, FaceRefLdg{P + f, pad});
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d2 = min_nn(d2, __shfl_xor_sync(0xffffffffu, d2, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = d2;
    __syncthreads();
    if (threadIdx.x == 0) {
        double r = red[0];
#pragma unroll
        for (int w = 1; w < kTile / 32; ++w) r = min_nn(r, red[w]);
        if (r < pos_inf()) atomicMin(objmin + T.obj, (unsigned long long)__double_as_longlong(r));
    }
}

// per object: band from the filter minimum and the object's header
__global__ void lt_band_kernel(QArgs a, uint64_t n_obj, const double* obj_stats, const unsigned long long* objmin,
                               double* band2, double* band, unsigned long long* D, unsigned long long* Pf) {
    const uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= n_obj) return;
    D[o] = Pf[o] = kNone;
    if (objmin[o] == kNone) {
        band2[o] = band[o] = -1.0;
        return;
    }
    const double m = sqrt(__longlong_as_double((long long)objmin[o]));
    const double b = m * (1.0 + kBandRel) + 2.0 * q_eta(load_query(a, 0), obj_stats + o * kObjStats, m);
    band[o] = b;
    band2[o] = b * b * (1.0 + 4e-16);
}

__global__ void __launch_bounds__(kTile) lt_verify_kernel(QArgs a, const Tile* tiles, const double* P, uint64_t pad,
                                                          int pass, const double* band2, unsigned long long* D,
                                                          unsigned long long* Pf, unsigned long long* ncand,
                                                          NearLog near) {
    const Tile T = tiles[blockIdx.x];
    const double b2 = band2[T.obj];
    if (b2 < 0.0 || threadIdx.x >= T.count) return;
    const uint64_t f = T.row0 + threadIdx.x;
    if (face_skipped(a, P, pad, f, T.obj)) return;
    const QueryRegs Q = load_query(a, 0);
    if (query_d2(Q, FaceRefLdg{P + f, pad}) > b2) return;
    const exact::tri t = face_tri(P, pad, f);
    const exact::v3 p0{Q.p0[0], Q.p0[1], Q.p0[2]}, p1{Q.p1[0], Q.p1[1], Q.p1[2]};
    const double d = Q.point ? exact::pt_tri(p0, t).d : exact::seg_tri(p0, p1, t).d;
    const unsigned long long e = (unsigned long long)__double_as_longlong(d);
    if (pass == 1) {
        atomicMin(D + T.obj, e);
        atomicAdd(ncand, 1ull);
        if (Q.point ? exact::near_area(t) : exact::near_degenerate_seg(p0, p1, t))
            near_log(near, T.obj, f - T.obj_row0);
    } else if (e == D[T.obj]) {
        atomicMin(Pf + T.obj, (unsigned long long)(f - T.obj_row0));
    }
}

__global__ void lt_check_kernel(QArgs a, uint64_t n_obj, const double* obj_stats, double* band2, double* band,
                                unsigned long long* D, unsigned long long* Pf, unsigned long long* retry) {
    const uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= n_obj) return;
    const double b = band[o];
    if (b < 0.0) {
        band2[o] = -1.0;
        return;
    }
    const QueryRegs Q = load_query(a, 0);
    const double* Bs = obj_stats + o * kObjStats;
    const unsigned long long d = D[o];
    const double m = d != kNone ? __longlong_as_double((long long)d) : 0.0;
    if (d != kNone && m + q_eta(Q, Bs, m) > b) {
        const double nb = m * (1.0 + kBandRel) + 2.0 * q_eta(Q, Bs, m);
        band[o] = nb;
        band2[o] = nb * nb * (1.0 + 4e-16);
        D[o] = Pf[o] = kNone;
        atomicAdd(retry, 1ull);
    } else {
        band2[o] = -1.0;
    }
}

// intersects: the q_hit_kernel cull (face box vs segment box +- tau, both
// endpoints strictly on one side of the face plane by tau), then the exact
// predicate; a tile is skipped once its object has a lower hit
__global__ void __launch_bounds__(kTile) lt_hit_kernel(QArgs a, const Tile* tiles, const double* P, uint64_t pad,
                                                       const double* obj_stats, unsigned long long* hitf,
                                                       unsigned long long* nexact, NearLog near) {
    const Tile T = tiles[blockIdx.x];
    const uint64_t rel0 = T.row0 - T.obj_row0;
    if (*(volatile unsigned long long*)(hitf + T.obj) < rel0 || threadIdx.x >= T.count) return;
    const uint64_t f = T.row0 + threadIdx.x;
    double p0[3], p1[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        p0[k] = __ldg(a.Q + (uint64_t)k * a.Qpad);
        p1[k] = __ldg(a.Q + (uint64_t)(3 + k) * a.Qpad);
    }
    const double* Bs = obj_stats + (uint64_t)T.obj * kObjStats;
    double ext = Bs[7], slo[3], shi[3], flo[3], fhi[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        ext = fmax(ext, fmax(fabs(p0[k]), fabs(p1[k])));
        slo[k] = fmin(p0[k], p1[k]), shi[k] = fmax(p0[k], p1[k]);
        flo[k] = __ldg(P + (uint64_t)(F_LO + k) * pad + f), fhi[k] = __ldg(P + (uint64_t)(F_HI + k) * pad + f);
    }
    if (seg_face_culled(p0, p1, slo, shi, flo, fhi, __ldg(P + (uint64_t)F_N * pad + f),
                        __ldg(P + (uint64_t)(F_N + 1) * pad + f), __ldg(P + (uint64_t)(F_N + 2) * pad + f),
                        __ldg(P + (uint64_t)F_C * pad + f), __ldg(P + (uint64_t)F_K * pad + f), kCullAbs * ext))
        return;
    atomicAdd(nexact, 1ull);
    const exact::tri t = face_tri(P, pad, f);
    const exact::v3 e0{p0[0], p0[1], p0[2]}, e1{p1[0], p1[1], p1[2]};
    if (exact::near_degenerate_seg(e0, e1, t)) near_log(near, T.obj, f - T.obj_row0);
    if (exact::seg_tri_hit(e0, e1, t)) atomicMin(hitf + T.obj, (unsigned long long)(f - T.obj_row0));
}

__global__ void lt_finalize_kernel(uint64_t n, const unsigned long long* D, const unsigned long long* Pf,
                                   double* dist, uint8_t* hit) {
    const uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= n) return;
    if (dist) dist[o] = Pf[o] == kNone || !D ? pos_inf() : __longlong_as_double((long long)D[o]);
    if (hit) hit[o] = Pf[o] != kNone;
}

}  // namespace

void run_literal_table(const Ctx& cx, int op, const QuerySet& q1, const Geom& B, double* dist, uint8_t* hit,
                       uint64_t* face) {
    const cudaStream_t st = cx.stream;
    tdb_stats& S = *cx.stats;
    std::memset(&S, 0, sizeof S);
    const uint64_t n_obj = B.n_obj, n_tiles = B.h_tiles.size();
    if (q1.n != 1) throw std::invalid_argument("one literal query expected");
    if (n_obj == 0) return;
    if (op == TDB_OP_INTERSECTS && q1.kind != kQuerySegments)
        throw std::invalid_argument("intersects takes a segment literal (batch.cpp:53-63)");
    std::vector<void*> mem;
    auto alloc = [&](size_t bytes) {
        void* p = nullptr;
        CK(cudaMallocAsync(&p, std::max<size_t>(1, bytes), st));
        mem.push_back(p);
        return p;
    };
    unsigned long long* ctr = (unsigned long long*)alloc(4 * sizeof(unsigned long long));
    CK(cudaMemsetAsync(ctr, 0, 4 * sizeof(unsigned long long), st));
    unsigned long long* D = (unsigned long long*)alloc(n_obj * sizeof(unsigned long long));
    unsigned long long* Pf = (unsigned long long*)alloc(n_obj * sizeof(unsigned long long));
    NearDev near;
    near.alloc(st);
    QArgs a{q1.planes, 1, q1.pad, q1.kind, B.planes, B.n_pad, B.n, 1, B.n, nullptr, nullptr, B.d_keep_deg};
    cudaEvent_t* ev = thread_events().e;
    CK(cudaEventRecord(ev[0], st));
    uint64_t launches = 0;
    int rounds = 0;
    if (n_tiles) {
        if (op == TDB_OP_INTERSECTS) {
            CK(cudaMemsetAsync(Pf, 0xff, n_obj * sizeof(unsigned long long), st));
            lt_hit_kernel<<<(unsigned)n_tiles, kTile, 0, st>>>(a, B.d_tiles, B.planes, B.n_pad, B.d_obj_stats, Pf,
                                                               ctr + 1, near.log);
            CK(cudaGetLastError());
            ++launches;
        } else {
            unsigned long long* objmin = (unsigned long long*)alloc(n_obj * sizeof(unsigned long long));
            double* band2 = (double*)alloc(n_obj * sizeof(double));
            double* band = (double*)alloc(n_obj * sizeof(double));
            CK(cudaMemsetAsync(objmin, 0xff, n_obj * sizeof(unsigned long long), st));
            const unsigned ob = (unsigned)((n_obj + 255) / 256);
            lt_filter_kernel<<<(unsigned)n_tiles, kTile, 0, st>>>(a, B.d_tiles, B.planes, B.n_pad, objmin);
            lt_band_kernel<<<ob, 256, 0, st>>>(a, n_obj, B.d_obj_stats, objmin, band2, band, D, Pf);
            launches += 2;
            for (rounds = 1; rounds <= 8; ++rounds) {
                for (int pass = 1; pass <= 2; ++pass) {
                    lt_verify_kernel<<<(unsigned)n_tiles, kTile, 0, st>>>(a, B.d_tiles, B.planes, B.n_pad, pass,
                                                                          band2, D, Pf, ctr, near.log);
                    ++launches;
                }
                CK(cudaMemsetAsync(ctr + 2, 0, sizeof(unsigned long long), st));
                lt_check_kernel<<<ob, 256, 0, st>>>(a, n_obj, B.d_obj_stats, band2, band, D, Pf, ctr + 2);
                ++launches;
                CK(cudaGetLastError());
                unsigned long long retry = 0;
                CK(cudaMemcpyAsync(&retry, ctr + 2, sizeof retry, cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                if (!retry) break;
            }
        }
    } else if (op == TDB_OP_INTERSECTS) {
        CK(cudaMemsetAsync(Pf, 0xff, n_obj * sizeof(unsigned long long), st));
    } else {
        CK(cudaMemsetAsync(D, 0xff, n_obj * sizeof(unsigned long long), st));
        CK(cudaMemsetAsync(Pf, 0xff, n_obj * sizeof(unsigned long long), st));
    }
    double* od = dist ? (double*)alloc(n_obj * sizeof(double)) : nullptr;
    uint8_t* oh = hit ? (uint8_t*)alloc(n_obj) : nullptr;
    lt_finalize_kernel<<<(unsigned)((n_obj + 255) / 256), 256, 0, st>>>(n_obj, op == TDB_OP_DISTANCE ? D : nullptr,
                                                                        Pf, od, oh);
    CK(cudaGetLastError());
    ++launches;
    CK(cudaEventRecord(ev[1], st));
    if (od) d2h(dist, od, n_obj * sizeof(double), st);
    if (oh) d2h(hit, oh, n_obj, st);
    if (face) d2h(face, Pf, n_obj * sizeof(uint64_t), st);
    unsigned long long hc[4] = {0, 0, 0, 0};
    CK(cudaMemcpyAsync(hc, ctr, sizeof hc, cudaMemcpyDeviceToHost, st));
    for (void* p : mem) CK(cudaFreeAsync(p, st));
    CK(cudaStreamSynchronize(st));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, ev[0], ev[1]));
    S.ms_total = ms;
    S.pairs = B.n;
    S.pairs_evaluated = B.n;
    S.items = n_tiles;
    S.candidates = hc[0];
    S.exact_pairs = hc[1];
    S.kernels = launches;
    S.rounds = rounds ? rounds : 1;
    near.fetch(st, cx.near);
    S.near_degenerate = cx.near->count;
}

namespace {

struct FaceIn {
    double q[6];
    double t9[9];
    int op, point;
};

// The reference's per-face result for one query (kernels.cpp:256-336 with
// their SurfaceParams / IntersectionParams), one thread.
__global__ void face_result_kernel(FaceIn in, tdb_face_result* out) {
    const exact::tri t{{in.t9[0], in.t9[1], in.t9[2]}, {in.t9[3], in.t9[4], in.t9[5]}, {in.t9[6], in.t9[7], in.t9[8]}};
    const exact::v3 p0{in.q[0], in.q[1], in.q[2]};
    const exact::v3 p1 = in.point ? p0 : exact::v3{in.q[3], in.q[4], in.q[5]};
    tdb_face_result r{};
    if (in.op == TDB_OP_DISTANCE) {
        exact::prm pr{0.0, 0.0, 0.0};
        const exact::res x = in.point ? exact::pt_tri(p0, t, &pr) : exact::seg_tri(p0, p1, t, &pr);
        r.distance = x.d;
        r.on_query[0] = x.a.x, r.on_query[1] = x.a.y, r.on_query[2] = x.a.z;
        r.on_face[0] = x.b.x, r.on_face[1] = x.b.y, r.on_face[2] = x.b.z;
        r.t = pr.t, r.u = pr.u, r.v = pr.v;
    } else {  // segment_triangle_intersect (kernels.cpp:318-336)
        const exact::v3 d = exact::sub(p1, p0);
        const exact::pierce_t x = exact::pierce(exact::sub(t.v1, t.v0), exact::sub(t.v2, t.v0), d, exact::sub(p0, t.v0));
        const double sl = exact::kSlack;
        if (x.ok && !(x.t < -sl || x.t > 1.0 + sl) && !(x.u < -sl || x.v < -sl || __dadd_rn(x.u, x.v) > 1.0 + sl)) {
            r.hit = 1;
            const exact::v3 pt = exact::add(p0, exact::scl(d, exact::clamp_unit(x.t)));
            r.point[0] = pt.x, r.point[1] = pt.y, r.point[2] = pt.z;
            r.t = x.t, r.u = x.u, r.v = x.v, r.w = __dsub_rn(__dsub_rn(1.0, x.u), x.v);
        }
    }
    *out = r;
}

}  // namespace

void run_face_result(const Ctx& cx, int op, int point, const double* q, const double* tri9, tdb_face_result* out) {
    FaceIn in{};
    std::copy(q, q + (point ? 3 : 6), in.q);
    std::copy(tri9, tri9 + 9, in.t9);
    in.op = op;
    in.point = point;
    tdb_face_result* d = nullptr;
    CK(cudaMallocAsync(&d, sizeof *d, cx.stream));
    face_result_kernel<<<1, 1, 0, cx.stream>>>(in, d);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, d, sizeof *out, cudaMemcpyDeviceToHost, cx.stream));
    CK(cudaFreeAsync(d, cx.stream));
    CK(cudaStreamSynchronize(cx.stream));
    std::memset(cx.stats, 0, sizeof *cx.stats);
    cx.stats->kernels = 1;
    cx.stats->pairs = 1;
}

}  // namespace tdb
