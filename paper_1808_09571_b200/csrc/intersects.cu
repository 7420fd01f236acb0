// ST_3DIntersects, mesh x mesh and table x mesh, with early exit.
//
// Semantics (oracle/tindb_oracle.c tri_tri_hit): a pair
// intersects iff any of the six directed edges passes the reference
// plane-piercing predicate segment_triangle_intersect (kernels.cpp:318-336,
// relative denominator eps 1e-12 and barycentric slack 1e-12; coplanar =>
// no hit). The object result is the lowest hit pair p = i*|B| + j
// (kernels.cpp:407-432).
//
// Culls (DESIGN.md 4.3 states and proves them; tdb_internal.h has the
// constants). They bound what the reference's OWN arithmetic can report,
// not only the exact geometry: its Cramer solve is noisy when a face is a
// sliver (noise ~ K = |e0||e1|/|N|) or an edge is nearly parallel to the
// other plane (noise up to 7.2e-3 D at its 1e-12 validity edge).
//   one-way : the other triangle's vertices beyond (kCullOne + kappa) D on
//             one side of this triangle's plane;
//   two-way : each triangle's vertices beyond (kCullTwo + kappa) D of the
//             other's plane (a t-rejection of all six edges);
//   apart   : object / tile / chunk boxes separated by kApart D.
// Everything else runs the bit-exact predicate (exact.cuh), so booleans and
// indices are the reference's (tests/test_gpu_parity.py, test_gpu_bounds.py).
//
// Layout: one warp per A-tile, each lane holds four rows (register blocking:
// one staged B face feeds four pair tests); B sub-tiles of kSBH faces are
// TMA bulk copies (15 SoA planes + 3 FP32 vertex planes) double-buffered on
// mbarriers. The hot test is the one-way cull of B's vertices against the
// row's plane, in FP32 first.
//
// Early exit: a warp skips its tile when the object's current lowest hit is
// below the tile's smallest pair index (kernels.cpp:413-415); a row stops at
// its first hit; an object whose AABB header is apart from B's is skipped
// whole.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "exact.cuh"
#include "runtime.h"
#include "tma.cuh"

namespace tdb {

namespace {

constexpr unsigned long long kNone = ~0ull;
constexpr int kHitPlanes = 15;  // V (9), N (3), C, DEG, K
__device__ __constant__ int kHitPlaneOf[kHitPlanes] = {0,   1,   2,       3,       4,   5,     6,  7,
                                                       8,   F_N, F_N + 1, F_N + 2, F_C, F_DEG, F_K};
enum { HS_V = 0, HS_N = 9, HS_C = 12, HS_DEG = 13, HS_K = 14 };
constexpr int kSBH = kHitGroup;    // B faces per staged sub-tile (one bounding sphere each)
constexpr int kRows = 4;           // A rows per lane
constexpr int kWarps = 4;          // tiles per CTA (one per warp)

struct HitArgs {
    const double* Ap;
    uint64_t An_pad;
    const Tile* tiles;
    uint64_t tile0, ntiles, row_lo, row_hi;
    const double* Bp;
    uint64_t Bn_pad, Bn, n_chunks, chunk;
    uint64_t obj0;
    const double* Astats;
    const double* Bstats;
    unsigned long long* objhit;
    unsigned long long* nexact;
    // CULL mode (null in FULL): per-tile and per-chunk AABBs
    const double* tile_aabb;
    const double* chunk_aabb;
    NearLog near;
    // FP32 pre-cull: B's vertices relative to its origin (3 float4 planes),
    // the origin, and a bound on |v - origin| over B
    const float* Bf;
    double ox, oy, oz, RB;
    const double4* Bsph;  // per kHitGroup B faces: bounding sphere (x, y, z, r)
};

__device__ __forceinline__ exact::tri load_tri(const double* P, uint64_t pad, uint64_t i) {
    double v[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) v[k] = __ldg(P + (uint64_t)(F_V + k) * pad + i);
    return exact::tri{{v[0], v[1], v[2]}, {v[3], v[4], v[5]}, {v[6], v[7], v[8]}};
}

// FP32 pre-cull: the same one-way test on h32 = n32 . (v - O) - c32 with
// |h32 - h| <= 6 * 2^-24 * (|v - O| + |c|) (roundings of n, v - O, c and
// three FMAs), so tau32 = kCull32 * (RB + |c|) + tau_one implies the FP64
// test separates too: the pre-cull never drops a pair the FP64 test keeps.
constexpr double kCull32 = 1e-6;

// all three h on one side, beyond tau: min > tau or max < -tau. (A NaN h
// needs an infinite input; the caller sets tau = +inf whenever FP32 could
// overflow, and then nothing is separated here.)
// Packed FP32 pairs (two rows at once): ptxas folds a {x, x} pack into an
// FFMA2 scalar-broadcast operand, so one FFMA2 does the FMA of two rows.
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
    unsigned long long d;
    asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(a), "f"(b));
    return d;
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ float lo2(unsigned long long x) { return __uint_as_float((unsigned)x); }
__device__ __forceinline__ float hi2(unsigned long long x) { return __uint_as_float((unsigned)(x >> 32)); }

__device__ __forceinline__ bool separated32(float h0, float h1, float h2, float tau) {
    return fminf(fminf(h0, h1), h2) > tau || fmaxf(fmaxf(h0, h1), h2) < -tau;
}

// all three h beyond tau on one common side (false for any NaN, or tau NaN)
__device__ __forceinline__ bool separated(double h0, double h1, double h2, double tau) {
    return (h0 > tau && h1 > tau && h2 > tau) || (h0 < -tau && h1 < -tau && h2 < -tau);
}

// The rest of the cull (the other one-way direction, then the two-way
// t-rejection) and the exact reference predicate: the rare path, out of line.
// h0..h2 are B's vertex heights above A's plane, kA / kB the faces' kappa.
static __device__ __noinline__ bool slow_pair(const double* Ap, uint64_t An_pad, uint64_t row, const double* sb,
                                              int j, double h0, double h1, double h2, double kA, double D,
                                              double abs_tol, const NearLog& near, unsigned long long obj,
                                              unsigned long long pair) {
    double av[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) av[k] = __ldg(Ap + (uint64_t)(F_V + k) * An_pad + row);
    const double bn0 = sb[(HS_N + 0) * kSBH + j], bn1 = sb[(HS_N + 1) * kSBH + j], bn2 = sb[(HS_N + 2) * kSBH + j],
                 bc = sb[HS_C * kSBH + j], kB = sb[HS_K * kSBH + j];
    const double g0 = fma(bn0, av[0], fma(bn1, av[1], fma(bn2, av[2], -bc)));
    const double g1 = fma(bn0, av[3], fma(bn1, av[4], fma(bn2, av[5], -bc)));
    const double g2 = fma(bn0, av[6], fma(bn1, av[7], fma(bn2, av[8], -bc)));
    if (separated(g0, g1, g2, (kCullOne + kB) * D + abs_tol)) return false;
    if (separated(g0, g1, g2, (kCullTwo + kB) * D + abs_tol) && separated(h0, h1, h2, (kCullTwo + kA) * D + abs_tol))
        return false;
    const double* bv = sb + HS_V * kSBH + j;
    const exact::tri ta{{av[0], av[1], av[2]}, {av[3], av[4], av[5]}, {av[6], av[7], av[8]}};
    const exact::tri tb{{bv[0], bv[kSBH], bv[2 * kSBH]}, {bv[3 * kSBH], bv[4 * kSBH], bv[5 * kSBH]},
                        {bv[6 * kSBH], bv[7 * kSBH], bv[8 * kSBH]}};
    if (exact::near_degenerate_pair(ta, tb)) near_log(near, obj, pair);
    return exact::tri_tri_hit(ta, tb);
}

__global__ void hit_init_kernel(unsigned long long* objhit, uint64_t nobj, unsigned long long* nex,
                                unsigned long long* near_count) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (objhit && i < nobj) objhit[i] = kNone;
    if (i == 0) *nex = 0, *near_count = 0;
}

#ifndef TDB_HIT_MINB
#define TDB_HIT_MINB 4  // 4 CTAs/SM (128 registers): 1.33e12 vs 1.14e12 pairs/s at 3 (scripts/variants_hit.sh)
#endif
__global__ void __launch_bounds__(32 * kWarps, TDB_HIT_MINB) hit_kernel(HitArgs a) {
    __shared__ alignas(128) double sm[2][kHitPlanes * kSBH];
    __shared__ alignas(128) float4 smf[2][3 * kSBH];
    __shared__ alignas(8) uint64_t bar[2];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t groups = (a.ntiles + kWarps - 1) / kWarps;
    const uint64_t item = blockIdx.x;
    const uint64_t grp = item / a.n_chunks, ch = item - grp * a.n_chunks;
    const uint64_t tl = grp * kWarps + warp;
    const bool has_tile = tl < a.ntiles;
    const Tile T = a.tiles[a.tile0 + (has_tile ? tl : a.ntiles - 1)];
    const uint64_t o = T.obj - a.obj0;
    const uint64_t b0 = ch * a.chunk, b1 = min(a.Bn, b0 + a.chunk);
    (void)groups;

    // per-object AABB header vs B's AABB, expanded by tau
    const double* As = a.Astats + (uint64_t)T.obj * kObjStats;
    const double* Bs = a.Bstats;
    double diag2 = 0.0;
    bool apart = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double lo = fmin(As[k], Bs[k]), hi = fmax(As[3 + k], Bs[3 + k]);
        diag2 += (hi - lo) * (hi - lo);
    }
    const double D = sqrt(diag2), abs_tol = kCullAbs * fmax(As[7], Bs[7]);
    const double tau_blk = (kCullOne + As[8]) * D + abs_tol;  // >= every live row's one-way margin
    const double gap = kApart * D + abs_tol;
#pragma unroll
    for (int k = 0; k < 3; ++k) apart |= (As[k] > Bs[3 + k] + gap) || (Bs[k] > As[3 + k] + gap);
    if (a.chunk_aabb) {  // CULL: the warp's tile box vs this item's B-chunk box
        const double* ta = a.tile_aabb + (a.tile0 + (has_tile ? tl : a.ntiles - 1)) * 6;
        const double* cb = a.chunk_aabb + ch * 6;
#pragma unroll
        for (int k = 0; k < 3; ++k) apart |= (ta[k] > cb[3 + k] + gap) || (cb[k] > ta[3 + k] + gap);
    }

    // this lane's rows: lane, lane+32, lane+64, lane+96 of the warp's tile
    double an[kRows][3], ac[kRows];
    uint64_t rowv[kRows];
    unsigned live = 0;  // bit r: row r still searching
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
        const uint32_t idx = lane + 32 * r;
        const uint64_t row = T.row0 + min(idx, T.count - 1);
        rowv[r] = row;
        const bool ok = has_tile && !apart && idx < T.count && row >= a.row_lo && row < a.row_hi &&
                        __ldg(a.Ap + (uint64_t)F_DEG * a.An_pad + row) == 0.0;
        live |= ok ? 1u << r : 0u;
#pragma unroll
        for (int k = 0; k < 3; ++k) an[r][k] = __ldg(a.Ap + (uint64_t)(F_N + k) * a.An_pad + row);
        ac[r] = __ldg(a.Ap + (uint64_t)F_C * a.An_pad + row);
    }
    // the rows' planes in B's FP32 frame: h = n . (v - O) - (c - n . O)
    float an32[kRows][3], ac32[kRows], tau32[kRows];
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
        const double cB = fma(-an[r][0], a.ox, fma(-an[r][1], a.oy, fma(-an[r][2], a.oz, ac[r])));
#pragma unroll
        for (int k = 0; k < 3; ++k) an32[r][k] = __double2float_rn(an[r][k]);
        ac32[r] = __double2float_rn(cB);
        const double kA = __ldg(a.Ap + (uint64_t)F_K * a.An_pad + rowv[r]);
        const double t32 = kCull32 * (a.RB + fabs(cB)) + (kCullOne + kA) * D + abs_tol;
        tau32[r] = a.RB + fabs(cB) < 1e30 ? __double2float_ru(t32) : __int_as_float(0x7f800000);  // +inf: no FP32 cull
    }
    static_assert(kRows % 2 == 0, "rows are packed in pairs");
    unsigned long long nq[kRows / 2][3], cq[kRows / 2];  // {row 2q, row 2q+1}
#pragma unroll
    for (int q = 0; q < kRows / 2; ++q) {
#pragma unroll
        for (int k = 0; k < 3; ++k) nq[q][k] = pk2(an32[2 * q][k], an32[2 * q + 1][k]);
        cq[q] = pk2(-ac32[2 * q], -ac32[2 * q + 1]);
    }
    const uint64_t Bn = a.Bn;
    auto row_pmin = [&](int r, uint64_t f0) { return (rowv[r] - T.obj_row0) * Bn + f0; };
    {  // a lower pair of this object already hit: nothing here can lower it
        const unsigned long long h = *(volatile unsigned long long*)(a.objhit + o);
        if (h != kNone) {
#pragma unroll
            for (int r = 0; r < kRows; ++r)
                if (h < row_pmin(r, b0)) live &= ~(1u << r);
        }
    }
    const bool cta_idle = __syncthreads_and(live == 0);
    if (cta_idle) return;

    const int nsub = (int)((b1 - b0 + kSBH - 1) / kSBH);
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto issue = [&](int s) {
        const int st = s & 1;
        const uint64_t f0 = b0 + (uint64_t)s * kSBH;
        const int cnt = (int)min((uint64_t)kSBH, b1 - f0);
        const uint32_t bytes = (uint32_t)(((cnt + 1) & ~1) * sizeof(double));
        const uint32_t fbytes = (uint32_t)(cnt * sizeof(float4));
        mbar_expect_tx(&bar[st], bytes * kHitPlanes + fbytes * 3);
#pragma unroll 1
        for (int f = 0; f < kHitPlanes; ++f)
            bulk_g2s(&sm[st][f * kSBH], a.Bp + (uint64_t)kHitPlaneOf[f] * a.Bn_pad + f0, bytes, &bar[st]);
#pragma unroll 1
        for (int f = 0; f < 3; ++f)
            bulk_g2s(&smf[st][f * kSBH], reinterpret_cast<const float4*>(a.Bf) + (uint64_t)f * a.Bn_pad + f0, fbytes,
                     &bar[st]);
    };
    if (threadIdx.x == 0) {
        issue(0);
        if (nsub > 1) issue(1);
    }
    unsigned long long nex = 0;
#pragma unroll 1
    for (int s = 0; s < nsub; ++s) {
        const int st = s & 1;
        mbar_wait(&bar[st], (uint32_t)((s >> 1) & 1));
        const uint64_t f0 = b0 + (uint64_t)s * kSBH;
        const int cnt = (int)min((uint64_t)kSBH, b1 - f0);
        const double* sb = sm[st];
        {
            const unsigned long long h = *(volatile unsigned long long*)(a.objhit + o);
            if (h != kNone) {
#pragma unroll
                for (int r = 0; r < kRows; ++r)
                    if (h < row_pmin(r, f0)) live &= ~(1u << r);
            }
        }
        // rows whose one-way margin clears the sub-tile's bounding sphere: every
        // face of it is culled one-way (the object-level kappa_max bounds the
        // row's; the slack covers the heights' rounding)
        unsigned bc = 0;
        {
            const double2* sp = reinterpret_cast<const double2*>(a.Bsph + f0 / kHitGroup);
            const double2 c01 = __ldg(sp), c2r = __ldg(sp + 1);
            const double reach = c2r.y * (1.0 + 1e-9) + tau_blk + 1e-12 * (fabs(c01.x) + fabs(c01.y) + fabs(c2r.x));
#pragma unroll
            for (int r = 0; r < kRows; ++r) {
                const double t = fma(an[r][0], c01.x, fma(an[r][1], c01.y, fma(an[r][2], c2r.x, -ac[r])));
                const double rr = reach + 1e-12 * fabs(ac[r]);
                bc |= (t > rr || t < -rr) ? 1u << r : 0u;
            }
        }
        if (__any_sync(0xffffffffu, (live & ~bc) != 0)) {
            const float4* fb = smf[st];
            const int* degw = reinterpret_cast<const int*>(sb + HS_DEG * kSBH) + 1;  // high words
#pragma unroll 1
            for (int j = 0; j < cnt; ++j) {
                if (degw[2 * j] != 0) continue;  // uniform
                const float4 V0 = fb[j], V1 = fb[kSBH + j], V2 = fb[2 * kSBH + j];  // 3 x LDS.128
                const float X0 = V0.x, Y0 = V0.y, Z0 = V0.z, X1 = V1.x, Y1 = V1.y, Z1 = V1.z;
                const float X2 = V2.x, Y2 = V2.y, Z2 = V2.z;
                bool sep[kRows];
#pragma unroll
                for (int q = 0; q < kRows / 2; ++q) {  // FP32 pre-cull, rows 2q and 2q+1 packed
                    const unsigned long long h0 =
                        ffma2(nq[q][0], pk2(X0, X0), ffma2(nq[q][1], pk2(Y0, Y0), ffma2(nq[q][2], pk2(Z0, Z0), cq[q])));
                    const unsigned long long h1 =
                        ffma2(nq[q][0], pk2(X1, X1), ffma2(nq[q][1], pk2(Y1, Y1), ffma2(nq[q][2], pk2(Z1, Z1), cq[q])));
                    const unsigned long long h2 =
                        ffma2(nq[q][0], pk2(X2, X2), ffma2(nq[q][1], pk2(Y2, Y2), ffma2(nq[q][2], pk2(Z2, Z2), cq[q])));
                    sep[2 * q] = separated32(lo2(h0), lo2(h1), lo2(h2), tau32[2 * q]);
                    sep[2 * q + 1] = separated32(hi2(h0), hi2(h1), hi2(h2), tau32[2 * q + 1]);
                }
                if (sep[0] & sep[1] & sep[2] & sep[3]) continue;  // the common case: all four culled
                unsigned need = 0;
#pragma unroll
                for (int r = 0; r < kRows; ++r) need |= sep[r] ? 0u : 1u << r;
                need &= live & ~bc;
                while (need) {  // rare: FP64 plane test, second plane, exact predicate
                    const int r = __ffs(need) - 1;
                    need &= need - 1;
                    const double* bv = sb + HS_V * kSBH + j;
                    const double h0 = fma(an[r][0], bv[0], fma(an[r][1], bv[kSBH], fma(an[r][2], bv[2 * kSBH], -ac[r])));
                    const double h1 =
                        fma(an[r][0], bv[3 * kSBH], fma(an[r][1], bv[4 * kSBH], fma(an[r][2], bv[5 * kSBH], -ac[r])));
                    const double h2 =
                        fma(an[r][0], bv[6 * kSBH], fma(an[r][1], bv[7 * kSBH], fma(an[r][2], bv[8 * kSBH], -ac[r])));
                    const double kA = __ldg(a.Ap + (uint64_t)F_K * a.An_pad + rowv[r]);
                    if (separated(h0, h1, h2, (kCullOne + kA) * D + abs_tol)) continue;
                    ++nex;
                    if (slow_pair(a.Ap, a.An_pad, rowv[r], sb, j, h0, h1, h2, kA, D, abs_tol, a.near, a.obj0 + o,
                                  row_pmin(r, f0 + j))) {
                        atomicMin(a.objhit + o, row_pmin(r, f0 + j));
                        live &= ~(1u << r);  // later j of this row only give larger p
                    }
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && s + 2 < nsub) issue(s + 2);
    }
    if (nex) atomicAdd(a.nexact, nex);
}

}  // namespace

namespace {
void run_intersects_batch(const Ctx& cx, const ASel& sel, const Geom& B, uint8_t* hit, uint64_t* pair);
}  // namespace

void run_intersects(const Ctx& cx, const ASel& sel, const Geom& B, uint8_t* hit, uint64_t* pair) {
    if (direct_eligible(sel, B, TDB_OP_INTERSECTS) && !cx.shared_hit) return run_intersects_direct(cx, sel, B, hit, pair);
    const uint64_t ntiles = sel.tile1 - sel.tile0;
    const uint64_t groups = (ntiles + kWarps - 1) / kWarps;
    const uint64_t chunk = pick_chunk(groups, B.n, cx.sms, 12, 256);
    const uint64_t n_chunks = (B.n + chunk - 1) / chunk;
    if (groups * n_chunks <= max_items() || groups <= 1) return run_intersects_batch(cx, sel, B, hit, pair);
    // too many items for one launch: tile batches in row order, lowest hit per object
    const uint64_t nobj = sel.obj1 - sel.obj0;
    for (uint64_t o = 0; o < nobj; ++o) {
        if (hit) hit[o] = 0;
        pair[o] = kNone;
    }
    tdb_stats tot{};
    NearHost near_all;
    const uint64_t per = std::max<uint64_t>(1, max_items() / n_chunks) * kWarps;
    for (const ASel& b : tile_batches(sel, per)) {
        // a batch whose lowest pair is above the best hit so far cannot lower it
        // (the hit may come from this selection's earlier batches or, through
        // a device group's shared word, from another member)
        if (nobj == 1 && pair[0] != kNone && pair[0] < std::max(sel.A->h_tiles[b.tile0].row0, sel.row_lo) * B.n) break;
        const uint64_t k = b.obj1 - b.obj0;
        std::vector<uint8_t> h(k);
        std::vector<uint64_t> p(k);
        run_intersects_batch(cx, b, B, h.data(), p.data());
        for (uint64_t o = 0; o < k; ++o) {
            const uint64_t g = b.obj0 - sel.obj0 + o;
            if (h[o] && p[o] < pair[g]) {
                pair[g] = p[o];
                if (hit) hit[g] = 1;
            }
        }
        const tdb_stats& s = *cx.stats;
        tot.ms_total += s.ms_total, tot.ms_filter += s.ms_filter, tot.ms_verify += s.ms_verify;
        tot.pairs += s.pairs, tot.items += s.items, tot.items_flagged += s.items_flagged;
        tot.candidates += s.candidates, tot.exact_pairs += s.exact_pairs, tot.kernels += s.kernels;
        tot.pairs_evaluated += s.pairs_evaluated, tot.near_degenerate += s.near_degenerate;
        tot.rounds = std::max(tot.rounds, s.rounds);
        near_all.count += cx.near->count;
        for (size_t e = 0; e < cx.near->entries.size() && near_all.entries.size() < 2 * kNearLogCap; e += 2) {
            near_all.entries.push_back(cx.near->entries[e]);
            near_all.entries.push_back(cx.near->entries[e + 1]);
        }
    }
    *cx.stats = tot;
    *cx.near = near_all;
}

namespace {
void run_intersects_batch(const Ctx& cx, const ASel& sel, const Geom& B, uint8_t* hit, uint64_t* pair) {
    const cudaStream_t st = cx.stream;
    const uint64_t nobj = sel.obj1 - sel.obj0;
    const uint64_t ntiles = sel.tile1 - sel.tile0;
    const uint64_t groups = (ntiles + kWarps - 1) / kWarps;
    const uint64_t chunk = pick_chunk(groups, B.n, cx.sms, 12, 256);
    const uint64_t n_chunks = (B.n + chunk - 1) / chunk;
    const uint64_t n_items = groups * n_chunks;
    tdb_stats& S = *cx.stats;
    std::memset(&S, 0, sizeof S);
    for (uint64_t o = 0; o < nobj; ++o) {
        if (hit) hit[o] = 0;
        pair[o] = kNone;
    }
    if (nobj == 0 || n_items == 0) return;
    const Geom& A = *sel.A;
    // one scratch allocation; its head is the result block copied back in one
    // piece: per-object lowest hit | exact-pair count | near-degenerate log
    size_t off = 0;
    auto piece = [&](size_t bytes) {
        const size_t o = off;
        off = (off + std::max<size_t>(bytes, 8) + 255) & ~size_t(255);
        return o;
    };
    const size_t o_hit = piece(nobj * 8), o_nex = piece(8), o_nc = piece(8), o_ne = piece(2 * kNearLogCap * 8);
    const size_t result_bytes = off;
    char* base = nullptr;
    CK(cudaMallocAsync(&base, off, st));
    unsigned long long* nex = (unsigned long long*)(base + o_nex);
    unsigned long long* near_count = (unsigned long long*)(base + o_nc);
    const NearLog nlog{near_count, (unsigned long long*)(base + o_ne)};
    // a device group's shared lowest-hit word (initialised by the group) or our own
    const bool shared = cx.shared_hit != nullptr && nobj == 1;
    unsigned long long* objhit = shared ? cx.shared_hit : (unsigned long long*)(base + o_hit);
    hit_init_kernel<<<(unsigned)((std::max<uint64_t>(nobj, 1) + 255) / 256), 256, 0, st>>>(
        shared ? nullptr : objhit, nobj, nex, near_count);
    CK(cudaGetLastError());
    // B's statistics: its one object's device header (a mesh), else a copy
    double* Bstats = B.n_obj == 1 ? B.d_obj_stats : nullptr;
    double* Bstats_copy = nullptr;
    if (!Bstats) {
        CK(cudaMallocAsync(&Bstats_copy, kObjStats * sizeof(double), st));
        CK(cudaMemcpyAsync(Bstats_copy, B.stats, kObjStats * sizeof(double), cudaMemcpyHostToDevice, st));
        Bstats = Bstats_copy;
    }
    geom_hit_spheres(B, st);  // B's sub-tile spheres, once per store
    EventPair& evs = thread_events();
    cudaEvent_t e0 = evs.e[0], e1 = evs.e[1], e2 = evs.e[2];
    double* caabb = nullptr;
    if (cx.mode == TDB_MODE_CULL) {
        CK(cudaMallocAsync(&caabb, n_chunks * 6 * sizeof(double), st));
        chunk_aabbs(B, chunk, caabb, st);
    }
    // |v - origin| over B <= the diagonal of B's AABB (the origin is a vertex of B)
    double rb = 0.0;
    for (int k = 0; k < 3; ++k) rb += (B.stats[3 + k] - B.stats[k]) * (B.stats[3 + k] - B.stats[k]);
    rb = std::sqrt(rb) * (1.0 + 1e-12);
    CK(cudaEventRecord(e0, st));
    hit_kernel<<<(unsigned)n_items, 32 * kWarps, 0, st>>>(HitArgs{A.planes, A.n_pad, A.d_tiles, sel.tile0, ntiles,
                                                                  sel.row_lo, sel.row_hi, B.planes, B.n_pad, B.n,
                                                                  n_chunks, chunk, sel.obj0, A.d_obj_stats, Bstats,
                                                                  objhit, nex, caabb ? A.d_tile_aabb : nullptr,
                                                                  caabb, nlog, B.fplanes, B.origin[0],
                                                                  B.origin[1], B.origin[2], rb, B.d_hsph});
    CK(cudaGetLastError());
    CK(cudaEventRecord(e1, st));
    thread_local std::vector<unsigned long long> hres;
    hres.resize(result_bytes / 8);
    CK(cudaMemcpyAsync(hres.data(), base, result_bytes, cudaMemcpyDeviceToHost, st));
    unsigned long long shared_best = kNone;
    if (shared) CK(cudaMemcpyAsync(&shared_best, objhit, sizeof shared_best, cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(e2, st));
    CK(cudaFreeAsync(base, st));
    if (Bstats_copy) CK(cudaFreeAsync(Bstats_copy, st));
    if (caabb) CK(cudaFreeAsync(caabb, st));
    CK(cudaStreamSynchronize(st));
    const unsigned long long* hp = shared ? &shared_best : hres.data() + o_hit / 8;
    for (uint64_t o = 0; o < nobj; ++o) {
        pair[o] = hp[o];
        if (hit) hit[o] = hp[o] != kNone;
    }
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    S.ms_filter = ms;
    CK(cudaEventElapsedTime(&ms, e0, e2));
    S.ms_total = ms;
    uint64_t pairs = 0;
    for (uint64_t t = sel.tile0; t < sel.tile1; ++t) {
        const Tile& T = A.h_tiles[t];
        const uint64_t lo = std::max(T.row0, sel.row_lo), hi = std::min(T.row0 + T.count, sel.row_hi);
        if (hi > lo) pairs += (hi - lo) * B.n;
    }
    S.pairs = pairs;
    S.items = n_items;
    S.exact_pairs = hres[o_nex / 8];
    S.pairs_evaluated = pairs;  // covered (early exit and culls are not subtracted)
    S.kernels = 2;
    S.rounds = 1;
    const unsigned long long nc = hres[o_nc / 8];
    cx.near->count = nc;
    cx.near->entries.assign(hres.data() + o_ne / 8, hres.data() + o_ne / 8 + 2 * std::min<uint64_t>(nc, kNearLogCap));
    S.near_degenerate = nc;
}

}  // namespace

}  // namespace tdb
