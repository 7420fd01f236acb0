// ST_3DDistance, mesh x mesh and table x mesh.
//
// Semantics (oracle/tindb_oracle.c tri_tri): the pair
// distance is the reference composition of segment_triangle_distance
// (kernels.cpp:256) over the six directed triangle edges; the object result
// is the minimum over pairs p = i*|B| + j with the lowest p on ties
// (kernels.cpp:359,368-376); degenerate faces are skipped.
//
// Pipeline per call (all on one stream, one host sync at the end):
//   1. filter_kernel   — the roofline kernel: every pair of every
//      (A-tile x B-chunk) item through the FP64 filter (fast_pair.cuh);
//      per-item min d~^2 and per-object atomicMin.
//   2. band_kernel     — per object, band = sqrt(min d~^2)(1+1e-9) + eta.
//   3. flag_kernel     — items whose min d~^2 lies inside the band.
//   4. verify_kernel   — re-scan flagged items; pairs inside the band get the
//      bit-exact composition (exact.cuh); pass 1 atomicMin of the exact
//      distance, pass 2 atomicMin of the pair index among exact ties.
//   5. check_kernel    — if an object's exact minimum lies outside its band
//      (the reference over-estimated every in-band pair), widen the band to
//      it and repeat 3-5 for that object. The result is then provably the
//      reference's: every pair left out has d_ref >= d_true - ulp > band >=
//      the reported minimum.
#include <algorithm>
#include <cstring>
#include <vector>

#include <cub/cub.cuh>

#include "exact.cuh"
#include "runtime.h"
#include "tma.cuh"

namespace tdb {

namespace {

constexpr unsigned long long kNone = ~0ull;

struct DistArgs {
    const double* Ap;
    uint64_t An_pad;
    const Tile* tiles;
    uint64_t tile0, row_lo, row_hi;
    const double* Bp;
    uint64_t Bn_pad, Bn, n_chunks, chunk;
    uint64_t obj0;
    double* itemmin;
    unsigned long long* objmin;
    // CULL mode (null in FULL): items in ascending order of their AABB lower
    // bound (squared), and the sorted bounds
    const unsigned long long* perm;
    const unsigned long long* lb2;
    unsigned long long* evaluated;  // pairs actually run through the filter
    // B's feature blocks (tdb_internal.h kFB) and the staged block capacity
    const double* Bfb;
    const uint4* Bfhdr;
    uint32_t stage;  // doubles per SMEM stage (>= every block's used doubles, even)
    const double4* Bsph;  // per block: bounding sphere of its vertices
};

__device__ __forceinline__ double warp_min_nn(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = min_nn(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
}

#ifndef TDB_FILTER_MINB
#define TDB_FILTER_MINB 3
#endif
// unroll factors of the vertex / face / edge candidate loops
#ifndef TDB_UV
#define TDB_UV 4
#endif
#ifndef TDB_UF
#define TDB_UF 2
#endif
#ifndef TDB_UE
#define TDB_UE 2
#endif
constexpr int kUV = TDB_UV, kUF = TDB_UF, kUE = TDB_UE;
// kEdges: also B's edges against each row's three edges (CULL mode, one
// kernel per item); FULL mode runs those in edge_kernel over A's distinct
// edges instead.
#ifndef TDB_FACE_MINB
#define TDB_FACE_MINB 4
#endif
static_assert(kFB <= 64, "the face loop's straddle mask is 64 bits");
// SMEM stages of filter_kernel: FULL keeps kFStages blocks in flight, each
// released per warp (an "empty" mbarrier per stage), so a warp whose rows meet
// straddling faces no longer holds the CTA at a per-block barrier: warps may
// drift kFStages - 2 blocks apart. CULL (whole blocks) keeps two.
#ifndef TDB_FSTAGES
#define TDB_FSTAGES 4
#endif
#ifndef TDB_FCHUNK_MAJOR
#define TDB_FCHUNK_MAJOR 1
#endif
template <bool kEdges>
constexpr int filter_stages() { return kEdges ? 2 : TDB_FSTAGES; }
template <bool kEdges>
__global__ void __launch_bounds__(kTile, kEdges ? TDB_FILTER_MINB : TDB_FACE_MINB) filter_kernel(DistArgs a) {
    constexpr int NS = filter_stages<kEdges>();
    static_assert(NS >= 2, "at least double buffering");
    extern __shared__ __align__(128) double dsm[];  // NS stages of a.stage doubles: one feature block each
    __shared__ alignas(8) uint64_t bar[NS];         // full: the stage's TMA transaction landed
    __shared__ alignas(8) uint64_t ebar[NS];        // empty: every warp is done with the stage
    __shared__ double red[kTile / 32];

    // FULL: CTAs in chunk-major order (TDB_FCHUNK_MAJOR), so the CTAs resident
    // at a time share one or two B chunks and read them from L2, not HBM (the
    // item index, and so every output, is the same either way)
    uint64_t item;
    if (a.perm) {
        item = a.perm[blockIdx.x];
    } else if (TDB_FCHUNK_MAJOR) {
        const uint64_t nt = gridDim.x / a.n_chunks, c = blockIdx.x / nt;
        item = (blockIdx.x - c * nt) * a.n_chunks + c;
    } else {
        item = blockIdx.x;
    }
    const uint64_t tl = item / a.n_chunks, ch = item - tl * a.n_chunks;
    const Tile T = a.tiles[a.tile0 + tl];
    if (a.perm) {  // CULL: no pair of this item can beat the object's current minimum
        __shared__ int skip;
        if (threadIdx.x == 0) {  // one read, so the whole CTA takes the same branch
            const unsigned long long lb = a.lb2[blockIdx.x];
            skip = lb > *(volatile unsigned long long*)(a.objmin + (T.obj - a.obj0));
            if (skip) a.itemmin[item] = __longlong_as_double((long long)lb);
        }
        __syncthreads();
        if (skip) return;
    }
    const uint32_t r = min(threadIdx.x, T.count - 1);
    const uint64_t row = T.row0 + r;
    bool active = threadIdx.x < T.count && row >= a.row_lo && row < a.row_hi;
    AFace A;
    load_aface(A, FaceRefLdg{a.Ap + row, a.An_pad});
    active = active && __ldg(a.Ap + (uint64_t)F_DEG * a.An_pad + row) == 0.0;

    // the item's B faces [b0, b1) are whole feature blocks (chunk % kFB == 0)
    const uint64_t b0 = ch * a.chunk, b1 = min(a.Bn, b0 + a.chunk);
    const uint64_t blk0 = b0 / kFB;
    const int nblk = (int)((b1 - b0 + kFB - 1) / kFB);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < NS; ++i) {
            mbar_init(&bar[i], 1);
            mbar_init(&ebar[i], kTile / 32);
        }
        mbar_fence_init();
    }
    __syncthreads();
    // per stage, beside the block's records: its header and bounds, staged by
    // the same TMA transaction (the consumers then never wait on global loads)
    __shared__ alignas(16) uint4 shdr[NS];
    __shared__ alignas(16) double4 ssph[NS];
    auto issue = [&](int s) {
        const int st = s % NS;
        const uint4 hb = __ldg(&a.Bfhdr[blk0 + s]);
        // CULL: the whole block; FULL: [face planes | vertices of faces |
        // distinct vertices] (the planes for the rare straddling faces: read
        // from L2 they stalled the warp, and the CTA at its barrier)
        const uint32_t bytes = (kEdges ? hb.w : (kFP + kFV) * hb.x + kVR * hb.y) * (uint32_t)sizeof(double);
        mbar_expect_tx(&bar[st], bytes + (uint32_t)sizeof(uint4) + (kEdges ? 0u : (uint32_t)sizeof(double4)));
        bulk_g2s(&shdr[st], &a.Bfhdr[blk0 + s], sizeof(uint4), &bar[st]);
        if (!kEdges) bulk_g2s(&ssph[st], a.Bsph + blk0 + s, sizeof(double4), &bar[st]);
        if (bytes) bulk_g2s(dsm + (size_t)st * a.stage, a.Bfb + (blk0 + s) * (uint64_t)kFBCap, bytes, &bar[st]);
    };
    if (threadIdx.x == 0)
        for (int s = 0; s < min(NS, nblk); ++s) issue(s);
    int best = kInfHi, hmin = kInfHi;
    bool pierce = false;
    // A's plane n.x = c, for the signs of B's vertex heights (the straddle
    // test; a sign is wrong only within rounding of the plane, where the
    // vertex / edge candidates already bound the pair)
    const double cA = dot3(A.n, A.v[0], A.v[1], A.v[2]);
    // A's bounding sphere (FULL): a FP32 centre near the centroid, the radius
    // to it rounded up. A B block whose sphere is apart from it holds no face
    // that A's triangle can meet, so no piercing (the straddle loop only
    // decides pierce_t in FULL mode).
    float sAx = 0.f, sAy = 0.f, sAz = 0.f, sAr = 0.f;
    if (!kEdges) {
        sAx = (float)((A.v[0] + A.v[3] + A.v[6]) * (1.0 / 3.0));
        sAy = (float)((A.v[1] + A.v[4] + A.v[7]) * (1.0 / 3.0));
        sAz = (float)((A.v[2] + A.v[5] + A.v[8]) * (1.0 / 3.0));
        double r2 = 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double dx = A.v[3 * k] - sAx, dy = A.v[3 * k + 1] - sAy, dz = A.v[3 * k + 2] - sAz;
            r2 = fmax(r2, fma(dx, dx, fma(dy, dy, dz * dz)));
        }
        sAr = __double2float_ru(sqrt(r2) * (1.0 + 1e-9));
    }
#pragma unroll 1
    for (int s = 0; s < nblk; ++s) {
        const int st = s % NS;
        mbar_wait(&bar[st], (uint32_t)((s / NS) & 1));
        const uint4 h = shdr[st];
        const double* base = dsm + (size_t)st * a.stage;
        const double* fp = base;                                // face planes
        const double* fv = base + kFP * h.x;                    // vertices of faces
        const double* vr = fv + kFV * h.x;                      // distinct vertices
        const double* er = vr + kVR * h.y;                      // distinct edges (CULL only)
        // B's distinct vertices against A's face
#pragma unroll kUV
        for (int j = 0; j < (int)h.y; ++j) {
            const double2 p0 = reinterpret_cast<const double2*>(vr + kVR * j)[0];
            const double pz = vr[kVR * j + 2];
            int hs;
            hmin = min(hmin, vertex_cand(A, p0.x, p0.y, pz, hs));
        }
        // B's faces: does B straddle A's plane? CULL runs A's vertices
        // against every face here; FULL runs them in vertex_kernel over A's
        // distinct vertices, and here only on the (rare) straddling faces, to
        // decide the piercing test: the face loop collects them in a mask
        // and stays branch-free.
        const double* fpl = fp;
        auto straddling = [&](int j) {  // A's vertices against face j (+ hmin in CULL), piercing test
            const double2* q = reinterpret_cast<const double2*>(fv + kFV * j);
            const double2 q0 = q[0], q1 = q[1], q4 = q[4];
            const double* pl = fpl + kFP * j;
            const double nb[3] = {pl[FP_N], pl[FP_N + 1], pl[FP_N + 2]};
            const double ub[3] = {pl[FP_U], pl[FP_U + 1], pl[FP_U + 2]};
            const double vb[3] = {pl[FP_W], pl[FP_W + 1], pl[FP_W + 2]};
            double w0[3];
            int hm = hmin;
            const bool sa = a_vertex_cand(A, q0.x, q0.y, q1.x, nb, ub, vb, hm, w0);
            if (kEdges) hmin = hm;
            return sa;
        };
        unsigned long long smask = 0;
        // FULL: no face of the block can straddle A's plane when the block's
        // bounding sphere lies beyond it (margins >> the rounding of the
        // heights below, so every face would test "no straddle" anyway)
        bool maybe = true;
        if (!kEdges) {
            const double4 sp = ssph[st];
            const double t = fabs(fma(A.n[0], sp.x, fma(A.n[1], sp.y, fma(A.n[2], sp.z, -cA))));
            maybe = !(t > sp.w * (1.0 + 1e-9) + 1e-9 * (fabs(sp.x) + fabs(sp.y) + fabs(sp.z) + fabs(cA) + sp.w));
            // the two bounding spheres apart (margin >> the rounding of d2)
            const double dx = sp.x - sAx, dy = sp.y - sAy, dz = sp.z - sAz;
            const double rr = (sp.w + sAr) * (1.0 + 1e-9) + 1e-9 * (fabs(sp.x) + fabs(sp.y) + fabs(sp.z));
            maybe = maybe && !(fma(dx, dx, fma(dy, dy, dz * dz)) > rr * rr);
        }
#pragma unroll kUF
        for (int j = 0; j < (maybe ? (int)h.x : 0); ++j) {
            const double2* q = reinterpret_cast<const double2*>(fv + kFV * j);
            const double2 q0 = q[0], q1 = q[1], q2 = q[2], q3 = q[3], q4 = q[4];
            const double g0 = fma(A.n[0], q0.x, fma(A.n[1], q0.y, fma(A.n[2], q1.x, -cA)));
            const double g1 = fma(A.n[0], q1.y, fma(A.n[1], q2.x, fma(A.n[2], q2.y, -cA)));
            const double g2 = fma(A.n[0], q3.x, fma(A.n[1], q3.y, fma(A.n[2], q4.x, -cA)));
            const int sor = __double2hiint(g0) | __double2hiint(g1) | __double2hiint(g2);
            const int sand = __double2hiint(g0) & __double2hiint(g1) & __double2hiint(g2);
            const bool sb = !(sor >= 0 || sand < 0);  // B straddles A's plane
            if (kEdges) {
                if (straddling(j) && sb)
                    pierce |= pierce_slow(a.Ap + row, a.An_pad, a.Bp + (uint64_t)__double_as_longlong(q4.y), a.Bn_pad);
            } else {
                smask |= (unsigned long long)sb << j;
            }
        }
        while (smask) {  // FULL, rare (B's face from the staged records)
            const int j = __ffsll((long long)smask) - 1;
            smask &= smask - 1;
            if (straddling(j)) pierce |= pierce_t(a.Ap + row, a.An_pad, FaceRec{fv + kFV * j, fp + kFP * j});
        }
        // B's distinct edges against A's edges (CULL; FULL: edge_kernel)
#pragma unroll kUE
        for (int j = 0; j < (kEdges ? (int)h.z : 0); ++j) {
            const double2* q = reinterpret_cast<const double2*>(er + kER * j);
            const double2 q0 = q[0], q1 = q[1], q2 = q[2], q3 = q[3];
            best = min(best, edge_cand(A, q0.x, q0.y, q1.x, q1.y, q2.x, q2.y, q3.x, q3.y));
        }
        // release the stage (each warp), then refill the one every warp
        // released NS - 2 blocks ago: block q + NS into q's buffer
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&ebar[st]);
        const int q = s - (NS - 2);
        if (threadIdx.x == 0 && q >= 0 && q + NS < nblk) {
            mbar_wait(&ebar[q % NS], (uint32_t)((q / NS) & 1));
            issue(q + NS);
        }
    }
    double m = __hiloint2double(pierce ? 0 : min(best, hmin_sq(hmin)), 0);
    if (!active || b1 <= b0) m = pos_inf();
    m = warp_min_nn(m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    const int rows_live = __syncthreads_count(active);
    if (threadIdx.x == 0) {
        double mm = red[0];
#pragma unroll
        for (int w = 1; w < kTile / 32; ++w) mm = min_nn(mm, red[w]);
        a.itemmin[item] = mm;
        atomicAdd(a.evaluated, (unsigned long long)rows_live * (b1 - b0));
        if (mm < pos_inf()) atomicMin(a.objmin + (T.obj - a.obj0), (unsigned long long)__double_as_longlong(mm));
    }
}

#ifndef TDB_EDGE_MINB
#define TDB_EDGE_MINB 3
#endif
#ifndef TDB_UEE
#define TDB_UEE 4
#endif
constexpr int kUEE = TDB_UEE;

struct EdgeArgs {
    const double* Ae;        // A edge entries (tdb_internal.h kAER)
    uint64_t e_lo, e_hi;     // the selection's entries
    uint64_t tile0, tile1;   // the selection's tiles
    const Tile* tiles;
    const double* Bfb;
    const uint4* Bfhdr;
    uint32_t stage;
    uint64_t Bn, n_chunks, chunk, obj0;
    unsigned long long* itemmin;  // the filter's item minima (non-negative doubles as u64)
    unsigned long long* objmin;
    const float4* Bse;            // B's super-block edges (FP32 records, kBER) and their per-group offsets
    const uint64_t* Bse_off;
    double ox, oy, oz;            // their origin
};

// An edge's minimum into the (tile, chunk) items of its tiles inside the
// selection and into its object.
__device__ __forceinline__ void edge_min_out(const EdgeArgs& a, uint64_t tile, uint64_t ch,
                                             unsigned long long bits) {
    const uint64_t t2[2] = {tile & 0xffffffffull, tile >> 32};  // the edge's tiles
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const uint64_t t = t2[q];
        if ((q == 1 && t == t2[0]) || t < a.tile0 || t >= a.tile1) continue;  // outside the selection
        atomicMin(a.itemmin + (t - a.tile0) * a.n_chunks + ch, bits);
        atomicMin(a.objmin + (a.tiles[t].obj - a.obj0), bits);
    }
}

// Edge/edge candidates of FULL mode: one A distinct edge per thread (kTile
// consecutive entries of A's edge tiles per CTA) against every distinct edge
// of the item's B chunk (staged per feature block by one TMA bulk copy).
// Each thread's minimum goes into the (tile, chunk) item of its edge's tile
// and its object: a pair's nine edge/edge candidates are among these, so the
// item minimum is the minimum over its pairs of pair_d2 (up to the edge
// direction of a shared edge). A tile partly outside
// [row_lo, row_hi) contributes all its edges: a lower item minimum only
// widens the band (check_kernel), never drops a pair. This FP64 kernel runs
// when the chunk is not a multiple of kBSuper; edge32_kernel otherwise.
#ifndef TDB_EDGE_APT
#define TDB_EDGE_APT 3
#endif
constexpr int kEdgeAPT = TDB_EDGE_APT;  // A edges per thread (a B edge loaded once feeds kEdgeAPT pairs)

__global__ void __launch_bounds__(kTile, TDB_EDGE_MINB) edge_kernel(EdgeArgs a) {
    extern __shared__ __align__(128) double dsm[];
    __shared__ alignas(8) uint64_t bar[2];
    const uint64_t et = blockIdx.x / a.n_chunks, ch = blockIdx.x - et * a.n_chunks;
    double Q[kEdgeAPT][8];
    uint64_t tile[kEdgeAPT];
    bool active[kEdgeAPT];
    int best[kEdgeAPT];
#pragma unroll
    for (int i = 0; i < kEdgeAPT; ++i) {
        const uint64_t e = a.e_lo + (et * kEdgeAPT + i) * kTile + threadIdx.x;
        active[i] = e < a.e_hi;
        const double2* q = reinterpret_cast<const double2*>(a.Ae + min(e, a.e_hi - 1) * kAER);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double2 v = __ldg(q + k);
            Q[i][2 * k] = v.x, Q[i][2 * k + 1] = v.y;
        }
        tile[i] = (uint64_t)__double_as_longlong(__ldg(reinterpret_cast<const double*>(q) + AR_TILE));
        best[i] = kInfHi;
    }

    const uint64_t b0 = ch * a.chunk, b1 = min(a.Bn, b0 + a.chunk);
    const uint64_t blk0 = b0 / kFB;
    const int nunits = (int)((b1 - b0 + kFB - 1) / kFB);
    __shared__ alignas(16) uint4 shdr[2];
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto issue = [&](int s) {
        const int st = s & 1;
        const uint4 hb = __ldg(&a.Bfhdr[blk0 + s]);
        const uint32_t bytes = (uint32_t)(kER * hb.z) * (uint32_t)sizeof(double);
        const double* src = a.Bfb + (blk0 + s) * (uint64_t)kFBCap + (kFP + kFV) * hb.x + kVR * hb.y;
        mbar_expect_tx(&bar[st], bytes + (uint32_t)sizeof(uint4));
        bulk_g2s(&shdr[st], &a.Bfhdr[blk0 + s], sizeof(uint4), &bar[st]);
        if (bytes) bulk_g2s(dsm + (size_t)st * a.stage, src, bytes, &bar[st]);
    };
    if (threadIdx.x == 0) {
        issue(0);
        if (nunits > 1) issue(1);
    }
#pragma unroll 1
    for (int s = 0; s < nunits; ++s) {
        const int st = s & 1;
        mbar_wait(&bar[st], (uint32_t)((s >> 1) & 1));
        const int ne = (int)shdr[st].z;
        const double* er = dsm + (size_t)st * a.stage;
#pragma unroll kUEE
        for (int j = 0; j < ne; ++j) {
            const double2* r = reinterpret_cast<const double2*>(er + (size_t)kER * j);
            const double2 p0 = r[0], p1 = r[1], p2 = r[2], p3 = r[3];
#pragma unroll
            for (int i = 0; i < kEdgeAPT; ++i)
                best[i] = min(best[i], edge_pair(Q[i][0], Q[i][1], Q[i][2], Q[i][3], Q[i][4], Q[i][5], Q[i][6], Q[i][7],
                                                 p0.x, p0.y, p1.x, p1.y, p2.x, p2.y, p3.x, p3.y));
        }
        __syncthreads();
        if (threadIdx.x == 0 && s + 2 < nunits) issue(s + 2);
    }
#pragma unroll
    for (int i = 0; i < kEdgeAPT; ++i)
        if (active[i] && best[i] < kInfHi)
            edge_min_out(a, tile[i], ch, (unsigned long long)__double_as_longlong(__hiloint2double(best[i], 0)));
}

// The same candidates on B's distinct edges per kBSuper faces (the chunk is a
// multiple of kBSuper), in FP32 (fast_pair.cuh edge_pair32; the band adds
// eta_f32): kEdge32APT A edges per thread, B's FP32 records streamed
// kEdgePiece per TMA stage (8 KB).
#ifndef TDB_E32_APT
#define TDB_E32_APT 4
#endif
#ifndef TDB_E32_MINB
#define TDB_E32_MINB 5
#endif
#ifndef TDB_UE32
#define TDB_UE32 2
#endif
// two A edges per packed FP32 pair (fast_pair.cuh edge_pair32x2; bit-identical values)
#ifndef TDB_E32_PACKED
#define TDB_E32_PACKED 1
#endif
constexpr int kEdge32APT = TDB_E32_APT;
constexpr int kUE32 = TDB_UE32;

__global__ void __launch_bounds__(kTile, TDB_E32_MINB) edge32_kernel(EdgeArgs a) {
    __shared__ alignas(128) float4 rec[2][2 * kEdgePiece];
    __shared__ alignas(8) uint64_t bar[2];
    const uint64_t et = blockIdx.x / a.n_chunks, ch = blockIdx.x - et * a.n_chunks;
    float Q[kEdge32APT][8];
    uint64_t tile[kEdge32APT];
    bool active[kEdge32APT];
    float best[kEdge32APT];
#pragma unroll
    for (int i = 0; i < kEdge32APT; ++i) {
        const uint64_t e = a.e_lo + (et * kEdge32APT + i) * kTile + threadIdx.x;
        active[i] = e < a.e_hi;
        const double* q = a.Ae + min(e, a.e_hi - 1) * kAER;
        const double2 v0 = __ldg(reinterpret_cast<const double2*>(q)), v1 = __ldg(reinterpret_cast<const double2*>(q) + 1),
                      v2 = __ldg(reinterpret_cast<const double2*>(q) + 2), v3 = __ldg(reinterpret_cast<const double2*>(q) + 3);
        Q[i][0] = (float)(v0.x - a.ox), Q[i][1] = (float)(v0.y - a.oy), Q[i][2] = (float)(v1.x - a.oz);
        Q[i][3] = (float)v1.y, Q[i][4] = (float)v2.x, Q[i][5] = (float)v2.y;
        Q[i][6] = (float)v3.x, Q[i][7] = (float)v3.y;
        tile[i] = (uint64_t)__double_as_longlong(__ldg(q + AR_TILE));
        best[i] = __int_as_float(0x7f800000);
    }

#if TDB_E32_PACKED
    static_assert(kEdge32APT % 2 == 0, "A edges in packed pairs");
    AEdge32x2 A2[kEdge32APT / 2];
#pragma unroll
    for (int i = 0; i < kEdge32APT / 2; ++i) {
        const float* x = Q[2 * i];
        const float* y = Q[2 * i + 1];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            A2[i].q[k] = pk2f(x[k], y[k]);
            A2[i].e[k] = pk2f(x[3 + k], y[3 + k]);
            A2[i].ne[k] = pk2f(-x[3 + k], -y[3 + k]);
        }
        A2[i].L = pk2f(x[6], y[6]);
        A2[i].il[0] = x[7], A2[i].il[1] = y[7];
    }
#endif

    const uint64_t b0 = ch * a.chunk, b1 = min(a.Bn, b0 + a.chunk);
    const uint64_t se0 = __ldg(a.Bse_off + b0 / kBSuper), se1 = __ldg(a.Bse_off + (b1 + kBSuper - 1) / kBSuper);
    const int nunits = (int)((se1 - se0 + kEdgePiece - 1) / kEdgePiece);
    auto unit_count = [&](int s) -> int { return (int)min((uint64_t)kEdgePiece, se1 - se0 - (uint64_t)s * kEdgePiece); };
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto issue = [&](int s) {
        const int st = s & 1;
        const uint32_t bytes = (uint32_t)unit_count(s) * 2u * (uint32_t)sizeof(float4);
        mbar_expect_tx(&bar[st], bytes);
        bulk_g2s(&rec[st][0], a.Bse + 2 * (se0 + (uint64_t)s * kEdgePiece), bytes, &bar[st]);
    };
    if (threadIdx.x == 0) {
        if (nunits > 0) issue(0);
        if (nunits > 1) issue(1);
    }
#pragma unroll 1
    for (int s = 0; s < nunits; ++s) {
        const int st = s & 1;
        mbar_wait(&bar[st], (uint32_t)((s >> 1) & 1));
        const int ne = unit_count(s);
        const float4* r = &rec[st][0];
#if TDB_E32_PACKED
#pragma unroll kUE32
        for (int j = 0; j < ne; ++j) {
            const float4 p0 = r[2 * j], p1 = r[2 * j + 1];
            const float nIL = -p1.w;
#pragma unroll
            for (int i = 0; i < kEdge32APT / 2; ++i) {
                float d0, d1;
                edge_pair32x2(A2[i], p0, p1, nIL, d0, d1);
                best[2 * i] = fminf(best[2 * i], d0);
                best[2 * i + 1] = fminf(best[2 * i + 1], d1);
            }
        }
#else
#pragma unroll kUE32
        for (int j = 0; j < ne; ++j) {
            const float4 p0 = r[2 * j], p1 = r[2 * j + 1];
#pragma unroll
            for (int i = 0; i < kEdge32APT; ++i) best[i] = fminf(best[i], edge_pair32(Q[i], p0, p1));
        }
#endif
        __syncthreads();
        if (threadIdx.x == 0 && s + 2 < nunits) issue(s + 2);
    }
#pragma unroll
    for (int i = 0; i < kEdge32APT; ++i)
        if (active[i] && best[i] < __int_as_float(0x7f800000)) edge_min_out(a, tile[i], ch, f32_as_f64_bits(best[i]));
}

struct VertArgs {
    const double* Av;        // A vertex entries (tdb_internal.h kAVR)
    uint64_t v_lo, v_hi;     // the selection's entries
    uint64_t tile0, tile1;
    const Tile* tiles;
    const double* Bfb;
    const uint4* Bfhdr;
    uint32_t stage;
    uint64_t Bn, n_chunks, chunk, obj0;
    unsigned long long* itemmin;
    unsigned long long* objmin;
};

#ifndef TDB_VERT_MINB
#define TDB_VERT_MINB 4
#endif
#ifndef TDB_UVF
#define TDB_UVF 4
#endif
constexpr int kUVF = TDB_UVF;

// Vertex/face candidates of FULL mode with A's vertices shared: one distinct
// vertex of an A tile per thread against every face of the item's B chunk
// (|h| when it projects inside; a_vertex_cand's arithmetic for that vertex).
// Minima into the (tile, chunk) items and objects as edge_kernel.
#ifndef TDB_VERT_APT
#define TDB_VERT_APT 2
#endif
constexpr int kVertAPT = TDB_VERT_APT;  // A vertices per thread (a B face loaded once feeds kVertAPT pairs)

__global__ void __launch_bounds__(kTile, TDB_VERT_MINB) vertex_kernel(VertArgs a) {
    extern __shared__ __align__(128) double dsm[];
    __shared__ alignas(8) uint64_t bar[2];
    __shared__ alignas(16) uint4 shdr[2];
    // chunk-major CTA order (as filter_kernel): resident CTAs share B chunks in L2
    const uint64_t n_vt = gridDim.x / a.n_chunks;
    const uint64_t ch = TDB_FCHUNK_MAJOR ? blockIdx.x / n_vt : blockIdx.x % a.n_chunks;
    const uint64_t vt = TDB_FCHUNK_MAJOR ? blockIdx.x - ch * n_vt : blockIdx.x / a.n_chunks;
    double ax[kVertAPT], ay[kVertAPT], az[kVertAPT];
    uint64_t tile[kVertAPT];
    bool active[kVertAPT];
    int hmin[kVertAPT];
#pragma unroll
    for (int i = 0; i < kVertAPT; ++i) {
        const uint64_t e = a.v_lo + (vt * kVertAPT + i) * kTile + threadIdx.x;
        active[i] = e < a.v_hi;
        const double2* q = reinterpret_cast<const double2*>(a.Av + min(e, a.v_hi - 1) * kAVR);
        const double2 q0 = __ldg(q), q1 = __ldg(q + 1);
        ax[i] = q0.x, ay[i] = q0.y, az[i] = q1.x;
        tile[i] = (uint64_t)__double_as_longlong(q1.y);
        hmin[i] = kInfHi;
    }

    const uint64_t b0 = ch * a.chunk, b1 = min(a.Bn, b0 + a.chunk);
    const uint64_t blk0 = b0 / kFB;
    const int nblk = (int)((b1 - b0 + kFB - 1) / kFB);
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto issue = [&](int s) {
        const int st = s & 1;
        const uint32_t bytes = (kFP + kFV) * __ldg(&a.Bfhdr[blk0 + s].x) * (uint32_t)sizeof(double);
        mbar_expect_tx(&bar[st], bytes + (uint32_t)sizeof(uint4));
        bulk_g2s(&shdr[st], &a.Bfhdr[blk0 + s], sizeof(uint4), &bar[st]);  // the header rides along
        if (bytes) bulk_g2s(dsm + (size_t)st * a.stage, a.Bfb + (blk0 + s) * (uint64_t)kFBCap, bytes, &bar[st]);
    };
    if (threadIdx.x == 0) {
        issue(0);
        if (nblk > 1) issue(1);
    }
#pragma unroll 1
    for (int s = 0; s < nblk; ++s) {
        const int st = s & 1;
        mbar_wait(&bar[st], (uint32_t)((s >> 1) & 1));
        const int nf = (int)shdr[st].x;
        const double2* fp = reinterpret_cast<const double2*>(dsm + (size_t)st * a.stage);  // face planes
        const double2* fv = fp + (kFP / 2) * nf;                                           // vertices of faces
#pragma unroll kUVF
        for (int j = 0; j < nf; ++j) {
            const double2* r = fp + (kFP / 2) * j;
            const double2 r0 = r[0], r1 = r[1], r2 = r[2], r3 = r[3], r4 = r[4];
            const double2 v0 = fv[(kFV / 2) * j], v1 = fv[(kFV / 2) * j + 1];
            const double nb[3] = {r0.x, r0.y, r1.x}, ub[3] = {r1.y, r2.x, r2.y}, vb[3] = {r3.x, r3.y, r4.x};
#pragma unroll
            for (int i = 0; i < kVertAPT; ++i) {
                const double wx = ax[i] - v0.x, wy = ay[i] - v0.y, wz = az[i] - v1.x;  // A_v - B_0
                const double h = dot3(nb, wx, wy, wz);
                const double u = dot3(ub, wx, wy, wz);
                const double v = dot3(vb, wx, wy, wz);
                hmin[i] = min(hmin[i], inside(u, v) ? (__double2hiint(h) & 0x7fffffff) : kInfHi);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && s + 2 < nblk) issue(s + 2);
    }
#pragma unroll
    for (int i = 0; i < kVertAPT; ++i)
        if (active[i] && hmin[i] < kInfHi) {
            const unsigned long long bits =
                (unsigned long long)__double_as_longlong(__hiloint2double(hmin_sq(hmin[i]), 0));
            const uint64_t t2[2] = {tile[i] & 0xffffffffull, tile[i] >> 32};  // the vertex's tiles
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const uint64_t t = t2[q];
                if ((q == 1 && t == t2[0]) || t < a.tile0 || t >= a.tile1) continue;  // outside the selection
                atomicMin(a.itemmin + (t - a.tile0) * a.n_chunks + ch, bits);
                atomicMin(a.objmin + (a.tiles[t].obj - a.obj0), bits);
            }
        }
}

struct BandArgs {
    const unsigned long long* objmin;
    const double* Astats;  // per object of A (absolute object index)
    const double* Bstats;  // aggregate of B (kObjStats doubles)
    uint64_t obj0, nobj;
    double* band2;
    double* band;
    unsigned long long* objD;
    unsigned long long* objP;
    double rB;  // the FP32 edge lists' origin radius (eta_f32) when they ran, else < 0
};

// eta(m) (tdb_internal.h) for objects A and B. The round is complete when the
// exact minimum D satisfies D + eta(D) <= band: every pair the reference can
// rank at or below D has d~ <= d_true + eta(d_true) <= D + eta(D) (eta grows
// with m), so it was flagged.
// With the FP32 edge lists (rB >= 0) eta_f32 is added: it bounds those
// candidates' excess (its supremum over d <= m, so the check still reads
// "D + eta(D) <= band").
__device__ __forceinline__ double band_eta(const double* As, const double* Bs, double m, double rB) {
    const double L = fmax(As[6], Bs[6]);
    const double e = band_eta_of(L, fmax(As[8], Bs[8]), fmax(As[7], Bs[7]), m);
    return rB >= 0.0 ? e + eta_f32(L, rB, m) : e;
}

__global__ void band_kernel(BandArgs a) {
    const uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= a.nobj) return;
    const unsigned long long e = a.objmin[o];
    a.objD[o] = kNone;
    a.objP[o] = kNone;
    if (e == kNone) {  // no non-degenerate pair
        a.band2[o] = -1.0;
        a.band[o] = -1.0;
        return;
    }
    const double m = sqrt(__longlong_as_double((long long)e));
    const double b = m * (1.0 + kBandRel) + 2.0 * band_eta(a.Astats + (a.obj0 + o) * kObjStats, a.Bstats, m, a.rB);
    a.band[o] = b;
    a.band2[o] = b * b * (1.0 + 4e-16);
}

struct FlagArgs {
    const Tile* tiles;
    uint64_t tile0, n_chunks, n_items, obj0;
    const double* itemmin;
    const double* band2;
    unsigned long long* list;
    unsigned long long* count;
};

__global__ void flag_kernel(FlagArgs a) {
    const uint64_t item = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (item >= a.n_items) return;
    const Tile T = a.tiles[a.tile0 + item / a.n_chunks];
    const double b2 = a.band2[T.obj - a.obj0];
    if (b2 >= 0.0 && a.itemmin[item] <= b2) a.list[atomicAdd(a.count, 1ull)] = item;
}

struct VerifyArgs {
    DistArgs d;
    const unsigned long long* list;
    const unsigned long long* count;
    int nsplit, pass;
    const double* band2;
    unsigned long long* objD;
    unsigned long long* objP;
    unsigned long long* ncand;
    NearLog near;
};

__device__ __forceinline__ exact::tri load_tri(const double* P, uint64_t pad, uint64_t i) {
    double v[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) v[k] = __ldg(P + (uint64_t)(F_V + k) * pad + i);
    return exact::tri{{v[0], v[1], v[2]}, {v[3], v[4], v[5]}, {v[6], v[7], v[8]}};
}

__global__ void __launch_bounds__(kTile) verify_kernel(VerifyArgs v) {
    const DistArgs& a = v.d;
    // split each flagged item's B range into nsplit parts, more when few
    // items are flagged so the grid stays busy (both passes see the same
    // count, hence the same split)
    const uint64_t count = *v.count;
    if (count == 0) return;
    const uint64_t nsplit = max((uint64_t)v.nsplit, min((uint64_t)a.chunk, (gridDim.x + count - 1) / count));
    const uint64_t units = count * nsplit;
    for (uint64_t w = blockIdx.x; w < units; w += gridDim.x) {
        const uint64_t item = v.list[w / nsplit];
        const uint64_t part = w % nsplit;
        const uint64_t tl = item / a.n_chunks, ch = item - tl * a.n_chunks;
        const Tile T = a.tiles[a.tile0 + tl];
        const uint32_t r = min(threadIdx.x, T.count - 1);
        const uint64_t row = T.row0 + r;
        bool active = threadIdx.x < T.count && row >= a.row_lo && row < a.row_hi;
        active = active && __ldg(a.Ap + (uint64_t)F_DEG * a.An_pad + row) == 0.0;
        AFace A;
        load_aface(A, FaceRefLdg{a.Ap + row, a.An_pad});
        const uint64_t c0 = ch * a.chunk, c1 = min(a.Bn, c0 + a.chunk);
        const uint64_t len = (c1 - c0 + nsplit - 1) / nsplit;
        const uint64_t b0 = min(c1, c0 + part * len), b1 = min(c1, b0 + len);
        const uint64_t o = T.obj - a.obj0;
        const double b2 = v.band2[o];
        const uint64_t i_loc = row - T.obj_row0;
        const int lane = threadIdx.x & 31;
        for (uint64_t j = b0; j < b1; ++j) {  // uniform across the CTA
            if (__ldg(a.Bp + (uint64_t)F_DEG * a.Bn_pad + j) != 0.0) continue;
            const double d2 = pair_d2(A, FaceRefLdg{a.Bp + j, a.Bn_pad}, a.Ap + row, a.An_pad);
            unsigned m = __ballot_sync(0xffffffffu, active && d2 <= b2);
            if (!m) continue;
            // the warp evaluates its band pairs one at a time, the exact
            // composition's six directed-edge seg_tri calls on six lanes
            // (exact::tri_tri, both triangles non-degenerate here), then the
            // same first-strict-minimum scan in the same order
            const exact::tri tb = load_tri(a.Bp, a.Bn_pad, j);
            while (m) {
                const int src = __ffs(m) - 1;
                m &= m - 1;
                const uint64_t rc = __shfl_sync(0xffffffffu, row, src);
                const exact::tri ta = load_tri(a.Ap, a.An_pad, rc);
                double dk = pos_inf();
                if (lane < 6) {
                    const exact::tri& s = lane < 3 ? ta : tb;
                    const exact::tri& t = lane < 3 ? tb : ta;
                    const int e = lane % 3;
                    const exact::v3 p0 = e == 0 ? s.v0 : e == 1 ? s.v1 : s.v2;
                    const exact::v3 p1 = e == 0 ? s.v1 : e == 1 ? s.v2 : s.v0;
                    dk = exact::seg_tri(p0, p1, t).d;
                }
                double x = pos_inf();
#pragma unroll
                for (int k = 0; k < 6; ++k) {
                    const double c = __shfl_sync(0xffffffffu, dk, k);
                    if (c < x) x = c;
                }
                if (lane == src) {
                    const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
                    if (v.pass == 1) {
                        atomicMin(v.objD + o, bits);
                        atomicAdd(v.ncand, 1ull);
                        if (exact::near_degenerate_pair(ta, tb)) near_log(v.near, a.obj0 + o, i_loc * a.Bn + j);
                    } else if (bits == v.objD[o]) {
                        atomicMin(v.objP + o, i_loc * a.Bn + j);
                    }
                }
            }
        }
    }
}

struct CheckArgs {
    uint64_t nobj, obj0;
    const double* Astats;
    const double* Bstats;
    double* band2;
    double* band;
    unsigned long long* objD;
    unsigned long long* objP;
    unsigned long long* retry;
    double rB;  // as BandArgs
};

// After a round: objects whose exact minimum lies outside the band get the
// band widened to it (and their exact state reset); the others stop.
__global__ void check_kernel(CheckArgs a) {
    const uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= a.nobj) return;
    const double b = a.band[o];
    if (b < 0.0) {
        a.band2[o] = -1.0;
        return;
    }
    const unsigned long long d = a.objD[o];
    // d == kNone: no pair fell in the band although the band contains the
    // filter minimum -> cannot happen unless every in-band pair evaluated to
    // NaN/inf; treat as done.
    const double* As = a.Astats + (a.obj0 + o) * kObjStats;
    const double m = d != kNone ? __longlong_as_double((long long)d) : 0.0;
    if (d != kNone && m + band_eta(As, a.Bstats, m, a.rB) > b) {
        const double nb = m * (1.0 + kBandRel) + 2.0 * band_eta(As, a.Bstats, m, a.rB);
        a.band[o] = nb;
        a.band2[o] = nb * nb * (1.0 + 4e-16);
        a.objD[o] = kNone;
        a.objP[o] = kNone;
        atomicAdd(a.retry, 1ull);
    } else {
        a.band2[o] = -1.0;  // final: do not re-flag
    }
}

// The winner's witness points: exact::tri_tri with its six directed-edge
// seg_tri calls on six lanes, then the same first-strict-minimum scan in the
// same order (so the same candidate wins as in the sequential composition).
__global__ void witness_kernel(const double* Ap, uint64_t An_pad, uint64_t obj_row0, const double* Bp,
                               uint64_t Bn_pad, uint64_t Bn, const unsigned long long* objP, double* out) {
    __shared__ exact::res c[6];
    const unsigned long long p = *objP;
    if (p == kNone) return;
    const uint64_t i = obj_row0 + p / Bn, j = p % Bn;
    const exact::tri a = load_tri(Ap, An_pad, i), b = load_tri(Bp, Bn_pad, j);
    const int k = threadIdx.x;
    if (k < 6) {
        const exact::tri& s = k < 3 ? a : b;
        const exact::tri& o = k < 3 ? b : a;
        const exact::v3 e0 = k % 3 == 0 ? s.v0 : k % 3 == 1 ? s.v1 : s.v2;
        const exact::v3 e1 = k % 3 == 0 ? s.v1 : k % 3 == 1 ? s.v2 : s.v0;
        c[k] = exact::seg_tri(e0, e1, o);
    }
    __syncthreads();
    if (k != 0 || exact::degenerate(a) || exact::degenerate(b)) return;
    exact::res best;
    best.d = pos_inf();
    best.a = best.b = exact::mk(0.0, 0.0, 0.0);
    for (int q = 0; q < 6; ++q)
        if (c[q].d < best.d) {
            best.d = c[q].d;
            best.a = q < 3 ? c[q].a : c[q].b;
            best.b = q < 3 ? c[q].b : c[q].a;
        }
    out[0] = best.a.x, out[1] = best.a.y, out[2] = best.a.z;
    out[3] = best.b.x, out[4] = best.b.y, out[5] = best.b.z;
}

// CULL: squared AABB distance between each item's A tile and B chunk (a lower
// bound of every pair distance in the item), as sortable u64 keys.
__global__ void item_bound_kernel(const double* __restrict__ tile_aabb, uint64_t tile0,
                                  const double* __restrict__ chunk_aabb, uint64_t n_chunks, uint64_t n_items,
                                  unsigned long long* __restrict__ keys, unsigned long long* __restrict__ vals) {
    const uint64_t item = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (item >= n_items) return;
    const uint64_t tl = item / n_chunks, ch = item - tl * n_chunks;
    const double* a = tile_aabb + (tile0 + tl) * 6;
    const double* b = chunk_aabb + ch * 6;
    double d2 = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double g = fmax(0.0, fmax(a[k] - b[3 + k], b[k] - a[3 + k]));
        d2 = fma(g, g, d2);
    }
    // round down: a bound, never above the true squared gap
    keys[item] = (unsigned long long)__double_as_longlong(__dmul_rd(d2, 1.0 - 1e-15));
    vals[item] = item;
}

template <class T>
T* dalloc(size_t n, cudaStream_t st) {
    T* p = nullptr;
    CK(cudaMallocAsync(&p, std::max<size_t>(1, n) * sizeof(T), st));
    return p;
}


// Device scratch of one call, one allocation. The result block (objD, objP,
// the witness, the counters, the near-degenerate log) is contiguous so one
// copy per round brings everything the host needs back.
struct DistScratch {
    unsigned long long* objD;  // result block begins here
    unsigned long long* objP;
    double* wit;
    unsigned long long* ctr;   // [1] candidates, [3] pairs evaluated; round r: [4+2r] flagged, [5+2r] retry
    unsigned long long* near_count;
    unsigned long long* near_entries;
    size_t result_bytes;       // objD .. near_entries end
    double* itemmin;
    unsigned long long* objmin;
    double* band2;
    double* band;
    unsigned long long* list;
    void* base;
};

constexpr int kMaxRounds = 8;                  // band widenings (2 in practice)
constexpr int kCtrSlots = 4 + 2 * kMaxRounds;  // per-round counters: no memsets between rounds

__global__ void dist_init_kernel(unsigned long long* objmin, uint64_t nobj, unsigned long long* ctr, double* wit,
                                 unsigned long long* near_count) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nobj) objmin[i] = kNone;
    if (i < kCtrSlots) ctr[i] = 0;
    if (i < 6) wit[i] = 0.0;
    if (i == 0) *near_count = 0;
}

}  // namespace

namespace {
void run_distance_batch(const Ctx& cx, const ASel& sel, const Geom& B, double* dist, uint64_t* pair,
                        double* witness6);
}  // namespace

void run_distance(const Ctx& cx, const ASel& sel, const Geom& B, double* dist, uint64_t* pair,
                  double* witness6) {
    if (direct_eligible(sel, B, TDB_OP_DISTANCE)) return run_distance_direct(cx, sel, B, dist, pair, witness6);
    const uint64_t ntiles = sel.tile1 - sel.tile0;
    const uint64_t chunk = pick_chunk(ntiles, B.n, cx.sms, 12, kFB);
    const uint64_t n_chunks = (B.n + chunk - 1) / chunk;
    if (ntiles * n_chunks <= max_items() || ntiles <= 1) return run_distance_batch(cx, sel, B, dist, pair, witness6);
    // too many items for one launch: tile batches, merged per object
    const uint64_t nobj = sel.obj1 - sel.obj0;
    for (uint64_t o = 0; o < nobj; ++o) dist[o] = pos_inf_h(), pair[o] = kNone;
    if (witness6) std::fill(witness6, witness6 + 6, 0.0);
    tdb_stats tot{};
    NearHost near_all;
    const uint64_t per = std::max<uint64_t>(1, max_items() / n_chunks);
    for (const ASel& b : tile_batches(sel, per)) {
        const uint64_t k = b.obj1 - b.obj0;
        std::vector<double> d(k), w6(6);
        std::vector<uint64_t> p(k);
        run_distance_batch(cx, b, B, d.data(), p.data(), witness6 ? w6.data() : nullptr);
        for (uint64_t o = 0; o < k; ++o) {
            const uint64_t g = b.obj0 - sel.obj0 + o;
            if (p[o] != kNone && (d[o] < dist[g] || (d[o] == dist[g] && p[o] < pair[g]))) {
                dist[g] = d[o];
                pair[g] = p[o];
                if (witness6 && nobj == 1) std::copy(w6.begin(), w6.end(), witness6);
            }
        }
        const tdb_stats& s = *cx.stats;
        tot.ms_total += s.ms_total, tot.ms_filter += s.ms_filter, tot.ms_verify += s.ms_verify;
        tot.pairs += s.pairs, tot.items += s.items, tot.items_flagged += s.items_flagged;
        tot.candidates += s.candidates, tot.kernels += s.kernels, tot.pairs_evaluated += s.pairs_evaluated;
        tot.near_degenerate += s.near_degenerate;
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
void run_distance_batch(const Ctx& cx, const ASel& sel, const Geom& B, double* dist, uint64_t* pair,
                        double* witness6) {
    const cudaStream_t st = cx.stream;
    const uint64_t nobj = sel.obj1 - sel.obj0;
    const uint64_t ntiles = sel.tile1 - sel.tile0;
    const uint64_t chunk = pick_chunk(ntiles, B.n, cx.sms, 12, kFB);
    const uint64_t n_chunks = (B.n + chunk - 1) / chunk;
    const uint64_t n_items = ntiles * n_chunks;
    for (uint64_t o = 0; o < nobj; ++o) {
        dist[o] = pos_inf_h();
        pair[o] = kNone;
    }
    if (witness6) std::fill(witness6, witness6 + 6, 0.0);
    tdb_stats& S = *cx.stats;
    std::memset(&S, 0, sizeof S);
    if (nobj == 0) return;
    if (n_items == 0) return;

    const Geom& A = *sel.A;
    geom_feature_blocks(B, st);  // B's feature blocks, once per store
    if (cx.mode != TDB_MODE_CULL) {
        geom_edge_tiles(A, st);  // A's super-tile lists, once per store
        if (pick_chunk(sel.tile1 - sel.tile0, B.n, cx.sms, 12, kFB) % kBSuper == 0) geom_bedges(B, st);  // B's, once
    }
    // ---- scratch layout (256-byte aligned pieces), one cudaMallocAsync
    DistScratch sc{};
    size_t off = 0;
    auto piece = [&](size_t bytes) {
        const size_t o = off;
        off = (off + std::max<size_t>(bytes, 8) + 255) & ~size_t(255);
        return o;
    };
    const size_t o_D = piece(nobj * 8), o_P = piece(nobj * 8), o_w = piece(6 * 8), o_c = piece(kCtrSlots * 8),
                 o_nc = piece(8), o_ne = piece(2 * kNearLogCap * 8);
    const size_t result_end = off;
    const size_t o_im = piece(n_items * 8), o_om = piece(nobj * 8), o_b2 = piece(nobj * 8), o_b = piece(nobj * 8),
                 o_l = piece(n_items * 8);
    char* base = dalloc<char>(off, st);
    sc.base = base;
    sc.objD = (unsigned long long*)(base + o_D);
    sc.objP = (unsigned long long*)(base + o_P);
    sc.wit = (double*)(base + o_w);
    sc.ctr = (unsigned long long*)(base + o_c);
    sc.near_count = (unsigned long long*)(base + o_nc);
    sc.near_entries = (unsigned long long*)(base + o_ne);
    sc.result_bytes = result_end;
    sc.itemmin = (double*)(base + o_im);
    sc.objmin = (unsigned long long*)(base + o_om);
    sc.band2 = (double*)(base + o_b2);
    sc.band = (double*)(base + o_b);
    sc.list = (unsigned long long*)(base + o_l);
    unsigned long long* const ctr = sc.ctr;
    const NearLog nlog{sc.near_count, sc.near_entries};
    // B's aggregate statistics: its one object's device header (a mesh), else a copy
    double* Bstats = B.n_obj == 1 ? B.d_obj_stats : nullptr;
    double* Bstats_copy = nullptr;
    if (!Bstats) {
        Bstats = Bstats_copy = dalloc<double>(kObjStats, st);
        CK(cudaMemcpyAsync(Bstats, B.stats, kObjStats * sizeof(double), cudaMemcpyHostToDevice, st));
    }
    dist_init_kernel<<<(unsigned)((std::max<uint64_t>(nobj, 8) + 255) / 256), 256, 0, st>>>(sc.objmin, nobj, ctr,
                                                                                           sc.wit, sc.near_count);
    CK(cudaGetLastError());

    EventPair& ev = thread_events();
    CK(cudaEventRecord(ev.e[0], st));
    uint64_t launches = 1;
    double rB = -1.0;  // >= 0 when the FP32 edge lists ran (band_eta adds eta_f32)
    unsigned long long *perm = nullptr, *lb2 = nullptr;
    void* cull_mem[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    if (cx.mode == TDB_MODE_CULL) {
        // branch and bound: items in ascending lower-bound order, skipped once
        // the bound exceeds the object's running minimum
        double* caabb = dalloc<double>(n_chunks * 6, st);
        unsigned long long* keys = dalloc<unsigned long long>(n_items, st);
        unsigned long long* vals = dalloc<unsigned long long>(n_items, st);
        lb2 = dalloc<unsigned long long>(n_items, st);
        perm = dalloc<unsigned long long>(n_items, st);
        chunk_aabbs(B, chunk, caabb, st);
        item_bound_kernel<<<(unsigned)((n_items + 255) / 256), 256, 0, st>>>(A.d_tile_aabb, sel.tile0, caabb,
                                                                            n_chunks, n_items, keys, vals);
        CK(cudaGetLastError());
        size_t tmp_bytes = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, lb2, vals, perm, (int)n_items, 0, 64, st));
        void* tmp = dalloc<unsigned char>(tmp_bytes, st);
        CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, lb2, vals, perm, (int)n_items, 0, 64, st));
        cull_mem[0] = caabb, cull_mem[1] = keys, cull_mem[2] = vals, cull_mem[3] = tmp;
        launches += 3;
    }
    // SMEM stages (128-byte aligned): a whole block (CULL), or only the part
    // each FULL kernel stages
    auto stage_of = [](uint32_t doubles) { return (std::max<uint32_t>(doubles, 2) + 15) & ~15u; };
    const uint32_t stage = stage_of(cx.mode == TDB_MODE_CULL ? B.fblock_max : B.fblock_max_pfv);
    const uint32_t stage_e = stage_of(B.fblock_max_e), stage_f = stage_of(B.fblock_max_f);
    const size_t smem = 2 * (size_t)stage * sizeof(double), smem_e = 2 * (size_t)stage_e * sizeof(double),
                 smem_f = 2 * (size_t)stage_f * sizeof(double);
    // per device (a device group calls from one thread per device); cheap
    CK(cudaFuncSetAttribute(filter_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            2 * kFBCap * (int)sizeof(double)));
    CK(cudaFuncSetAttribute(filter_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            filter_stages<false>() * kFBCap * (int)sizeof(double)));
    CK(cudaFuncSetAttribute(edge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            2 * kFBCap * (int)sizeof(double)));
    CK(cudaFuncSetAttribute(vertex_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            2 * kFBCap * (int)sizeof(double)));
    DistArgs da{A.planes, A.n_pad, A.d_tiles, sel.tile0, sel.row_lo, sel.row_hi, B.planes, B.n_pad, B.n,
                n_chunks, chunk, sel.obj0, sc.itemmin, sc.objmin, perm, lb2, ctr + 3, B.fblocks, B.d_fhdr, stage,
                B.d_fsph};
    if (cx.mode == TDB_MODE_CULL) {
        filter_kernel<true><<<(unsigned)n_items, kTile, smem, st>>>(da);
        CK(cudaGetLastError());
    } else {
        filter_kernel<false><<<(unsigned)n_items, kTile, filter_stages<false>() * (size_t)stage * sizeof(double), st>>>(da);
        CK(cudaGetLastError());
        // entries are ordered by their first tile: those of tiles [tile0, tile1)
        // lie in [first tile >= tile0 - span, first tile < tile1), span = the
        // largest (second - first tile) of tile0's super-tile
        const uint64_t st0 = A.h_tile_st[sel.tile0], t_st = A.h_st_tile0[st0];
        auto lo_tile = [&](uint32_t span) { return std::max<uint64_t>(t_st, sel.tile0 >= span ? sel.tile0 - span : 0); };
        const uint64_t v_lo = A.h_tile_voff[lo_tile(A.h_st_vspan[st0])], v_hi = A.h_tile_voff[sel.tile1];
        const uint64_t n_vt = (v_hi - v_lo + kTile * kVertAPT - 1) / (kTile * kVertAPT);
        if (n_vt) {
            vertex_kernel<<<(unsigned)(n_vt * n_chunks), kTile, smem_f, st>>>(
                VertArgs{A.averts, v_lo, v_hi, sel.tile0, sel.tile1, A.d_tiles, B.fblocks, B.d_fhdr, stage_f, B.n,
                         n_chunks, chunk,
                         sel.obj0, (unsigned long long*)sc.itemmin, sc.objmin});
            CK(cudaGetLastError());
            ++launches;
        }
        // (entries reaching back into tiles before tile0 are evaluated too;
        // the kernels attribute only to tiles inside the selection)
        const uint64_t e_lo = A.h_tile_eoff[lo_tile(A.h_st_espan[st0])], e_hi = A.h_tile_eoff[sel.tile1];
        // B's edges per kBSuper faces in FP32 when the chunk allows (fewer edge
        // pairs; coordinates within 1e15 so no FP32 value overflows), else per
        // feature block in FP64
        const bool super = chunk % kBSuper == 0 && B.d_bseoff && std::max(A.stats[7], B.stats[7]) < 1e15;
        const int apt = super ? kEdge32APT : kEdgeAPT;
        const uint64_t n_et = (e_hi - e_lo + (uint64_t)kTile * apt - 1) / ((uint64_t)kTile * apt);
        if (n_et) {
            const EdgeArgs ea{A.aedges, e_lo, e_hi, sel.tile0, sel.tile1, A.d_tiles, B.fblocks, B.d_fhdr, stage_e,
                              B.n, n_chunks, chunk, sel.obj0, (unsigned long long*)sc.itemmin, sc.objmin, B.bedges,
                              B.d_bseoff, B.bse_org[0], B.bse_org[1], B.bse_org[2]};
            if (super) {
                edge32_kernel<<<(unsigned)(n_et * n_chunks), kTile, 0, st>>>(ea);
                rB = B.bse_rB;
            } else {
                edge_kernel<<<(unsigned)(n_et * n_chunks), kTile, smem_e, st>>>(ea);
            }
            CK(cudaGetLastError());
            ++launches;
        }
    }
    CK(cudaEventRecord(ev.e[1], st));
    ++launches;

    const unsigned ob = (unsigned)((nobj + 255) / 256);
    band_kernel<<<ob, 256, 0, st>>>(BandArgs{sc.objmin, A.d_obj_stats, Bstats, sel.obj0, nobj, sc.band2, sc.band,
                                             sc.objD, sc.objP, rB});
    CK(cudaGetLastError());
    ++launches;

    const int nsplit = 16;
    const unsigned vgrid = (unsigned)(cx.sms * 8);
    const bool want_witness = witness6 && nobj == 1;
    // host copy of the result block (pinned per thread, grown on demand)
    thread_local std::vector<unsigned long long> hres;
    hres.resize(sc.result_bytes / 8);
    unsigned long long* h_ctr = hres.data() + o_c / 8;
    int rounds = 0;
    unsigned long long flagged_total = 0;
    for (;;) {
        ++rounds;
        unsigned long long* const flagged = ctr + 4 + 2 * (rounds - 1);  // zeroed by dist_init_kernel
        unsigned long long* const retry = flagged + 1;
        flag_kernel<<<(unsigned)((n_items + 255) / 256), 256, 0, st>>>(
            FlagArgs{A.d_tiles, sel.tile0, n_chunks, n_items, sel.obj0, sc.itemmin, sc.band2, sc.list, flagged});
        CK(cudaGetLastError());
        for (int pass = 1; pass <= 2; ++pass) {
            verify_kernel<<<vgrid, kTile, 0, st>>>(
                VerifyArgs{da, sc.list, flagged, nsplit, pass, sc.band2, sc.objD, sc.objP, ctr + 1, nlog});
            CK(cudaGetLastError());
        }
        check_kernel<<<ob, 256, 0, st>>>(CheckArgs{nobj, sel.obj0, A.d_obj_stats, Bstats, sc.band2, sc.band,
                                                   sc.objD, sc.objP, retry, rB});
        CK(cudaGetLastError());
        launches += 4;
        if (want_witness) {  // for this round's winner; recomputed if the band widens
            const Tile& t0 = A.h_tiles[sel.tile0];
            witness_kernel<<<1, 32, 0, st>>>(A.planes, A.n_pad, t0.obj_row0, B.planes, B.n_pad, B.n, sc.objP,
                                             sc.wit);
            CK(cudaGetLastError());
            ++launches;
        }
        CK(cudaEventRecord(ev.e[2], st));  // end of the device work (the last round's record stands)
        CK(cudaMemcpyAsync(hres.data(), base, sc.result_bytes, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        flagged_total += h_ctr[4 + 2 * (rounds - 1)];
        if (h_ctr[5 + 2 * (rounds - 1)] == 0 || rounds >= kMaxRounds) break;
    }
    CK(cudaFreeAsync(base, st));
    for (void* p : {(void*)Bstats_copy, (void*)perm, (void*)lb2, cull_mem[0], cull_mem[1], cull_mem[2], cull_mem[3]})
        if (p) CK(cudaFreeAsync(p, st));
    const unsigned long long* hD = hres.data() + o_D / 8;
    const unsigned long long* hP = hres.data() + o_P / 8;
    for (uint64_t o = 0; o < nobj; ++o) {
        if (hP[o] != kNone) {
            double d;
            std::memcpy(&d, &hD[o], sizeof d);
            dist[o] = d;
            pair[o] = hP[o];
        }
    }
    if (want_witness) std::memcpy(witness6, hres.data() + o_w / 8, 6 * sizeof(double));
    CK(cudaEventSynchronize(ev.e[2]));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, ev.e[0], ev.e[1]));
    S.ms_filter = ms;
    CK(cudaEventElapsedTime(&ms, ev.e[1], ev.e[2]));
    S.ms_verify = ms;
    CK(cudaEventElapsedTime(&ms, ev.e[0], ev.e[2]));
    S.ms_total = ms;
    uint64_t pairs = 0;
    for (uint64_t t = sel.tile0; t < sel.tile1; ++t) {
        const Tile& T = A.h_tiles[t];
        const uint64_t lo = std::max(T.row0, sel.row_lo), hi = std::min(T.row0 + T.count, sel.row_hi);
        if (hi > lo) pairs += (hi - lo) * B.n;
    }
    S.pairs = pairs;
    S.items = n_items;
    S.items_flagged = flagged_total;
    S.candidates = h_ctr[1];
    S.kernels = launches;
    S.pairs_evaluated = h_ctr[3];
    S.rounds = rounds;
    // near-degenerate log: came back with the result block
    const unsigned long long nc = hres[o_nc / 8];
    cx.near->count = nc;
    cx.near->entries.assign(hres.data() + o_ne / 8, hres.data() + o_ne / 8 + 2 * std::min<uint64_t>(nc, kNearLogCap));
    S.near_degenerate = nc;
}

}  // namespace

}  // namespace tdb
