// ST_3DIntersects, mesh x mesh and table x mesh, with early exit.
//
// Semantics (oracle/tindb_oracle.c tri_tri_hit): a pair
// intersects iff any of the six directed edges passes the reference
// plane-piercing predicate segment_triangle_intersect (kernels.cpp:318-336,
// relative denominator eps 1e-12 and barycentric slack 1e-12; coplanar =>
// no hit). The object result is the lowest hit pair p = i*|B| + j
// (kernels.cpp:407-432).
//
// Per pair the kernel first runs a conservative separating-plane test in
// FP64: if all three vertices of one triangle lie strictly on one side of
// the other's plane by more than tau (tdb_internal.h: 1e-10 x diag of the
// pair's bounding box + 1e-13 x max |coord|, >= 30x the reference
// predicate's worst rounding of t at that separation), no directed edge can
// pass the reference predicate. Survivors run
// the bit-exact predicate (exact.cuh), so booleans and indices are the
// reference's.
//
// Early exit: an item is skipped when the object's current lowest hit is
// below the item's smallest pair index (kernels.cpp:413-415), and an object
// whose AABB is separated from B's by more than tau is skipped whole (the
// per-object AABB header).
#include <algorithm>
#include <cstring>
#include <vector>

#include "exact.cuh"
#include "runtime.h"
#include "tma.cuh"

namespace tdb {

namespace {

constexpr unsigned long long kNone = ~0ull;
// staged B planes: V (0..8), N (24..26), C (27) -> copy planes [0,9) and [24,28), plus DEG
constexpr int kHitPlanes = 14;
__device__ __constant__ int kHitPlaneOf[kHitPlanes] = {0, 1, 2, 3, 4, 5, 6, 7, 8, F_N, F_N + 1, F_N + 2, F_C, F_DEG};
enum { HS_V = 0, HS_N = 9, HS_C = 12, HS_DEG = 13 };

struct HitArgs {
    const double* Ap;
    uint64_t An_pad;
    const Tile* tiles;
    uint64_t tile0, row_lo, row_hi;
    const double* Bp;
    uint64_t Bn_pad, Bn, n_chunks;
    uint64_t obj0;
    const double* Astats;
    const double* Bstats;
    unsigned long long* objhit;
    unsigned long long* nexact;
};

__device__ __forceinline__ exact::tri load_tri(const double* P, uint64_t pad, uint64_t i) {
    double v[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) v[k] = __ldg(P + (uint64_t)(F_V + k) * pad + i);
    return exact::tri{{v[0], v[1], v[2]}, {v[3], v[4], v[5]}, {v[6], v[7], v[8]}};
}

// all three |h| > tau with one common sign
__device__ __forceinline__ bool separated(double h0, double h1, double h2, double tau) {
    const double q0 = fabs(h0) - tau, q1 = fabs(h1) - tau, q2 = fabs(h2) - tau;
    const int s0 = __double2hiint(h0), s1 = __double2hiint(h1), s2 = __double2hiint(h2);
    const int same = (s0 ^ s1) | (s0 ^ s2);
    return (same | __double2hiint(q0) | __double2hiint(q1) | __double2hiint(q2)) >= 0 &&
           q0 != 0.0 && q1 != 0.0 && q2 != 0.0;
}

__global__ void __launch_bounds__(kTile, 4) hit_kernel(HitArgs a) {
    __shared__ alignas(128) double sm[2][kHitPlanes * kSB];
    __shared__ alignas(8) uint64_t bar[2];

    const uint64_t item = blockIdx.x;
    const uint64_t tl = item / a.n_chunks, ch = item - tl * a.n_chunks;
    const Tile T = a.tiles[a.tile0 + tl];
    const uint64_t o = T.obj - a.obj0;
    const uint64_t b0 = ch * kChunk, b1 = min(a.Bn, b0 + kChunk);
    const uint64_t first_row = max(T.row0, a.row_lo);
    const uint64_t pmin = (first_row - T.obj_row0) * a.Bn + b0;
    if (*(volatile unsigned long long*)(a.objhit + o) < pmin) return;  // a lower pair already hit

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
    const double tau = kCullDiag * sqrt(diag2) + kCullAbs * fmax(As[7], Bs[7]);
#pragma unroll
    for (int k = 0; k < 3; ++k) apart |= (As[k] > Bs[3 + k] + tau) || (Bs[k] > As[3 + k] + tau);
    if (apart) return;

    const uint32_t r = min(threadIdx.x, T.count - 1);
    const uint64_t row = T.row0 + r;
    bool active = threadIdx.x < T.count && row >= a.row_lo && row < a.row_hi;
    active = active && __ldg(a.Ap + (uint64_t)F_DEG * a.An_pad + row) == 0.0;
    double av[9], an[3], ac;
#pragma unroll
    for (int k = 0; k < 9; ++k) av[k] = __ldg(a.Ap + (uint64_t)(F_V + k) * a.An_pad + row);
#pragma unroll
    for (int k = 0; k < 3; ++k) an[k] = __ldg(a.Ap + (uint64_t)(F_N + k) * a.An_pad + row);
    ac = __ldg(a.Ap + (uint64_t)F_C * a.An_pad + row);
    const uint64_t i_loc = row - T.obj_row0;
    bool done = !active;

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
        mbar_expect_tx(&bar[st], bytes * kHitPlanes);
#pragma unroll 1
        for (int f = 0; f < kHitPlanes; ++f)
            bulk_g2s(&sm[st][f * kSB], a.Bp + (uint64_t)kHitPlaneOf[f] * a.Bn_pad + f0, bytes, &bar[st]);
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
        const uint64_t f0 = b0 + (uint64_t)s * kSB;
        const int cnt = (int)min((uint64_t)kSB, b1 - f0);
        const double* sb = sm[st];
        // stop rows whose smallest remaining pair cannot beat the object's hit
        if (!done && *(volatile unsigned long long*)(a.objhit + o) < i_loc * a.Bn + f0) done = true;
        if (!__syncthreads_and(done)) {
#pragma unroll 1
            for (int j = 0; j < cnt; ++j) {
                if (sb[HS_DEG * kSB + j] != 0.0) continue;
                if (done) continue;
                const double* bv = sb + HS_V * kSB + j;
                const double h0 = fma(an[0], bv[0], fma(an[1], bv[kSB], fma(an[2], bv[2 * kSB], -ac)));
                const double h1 = fma(an[0], bv[3 * kSB], fma(an[1], bv[4 * kSB], fma(an[2], bv[5 * kSB], -ac)));
                const double h2 = fma(an[0], bv[6 * kSB], fma(an[1], bv[7 * kSB], fma(an[2], bv[8 * kSB], -ac)));
                if (separated(h0, h1, h2, tau)) continue;
                const double bn0 = sb[(HS_N + 0) * kSB + j], bn1 = sb[(HS_N + 1) * kSB + j],
                             bn2 = sb[(HS_N + 2) * kSB + j], bc = sb[HS_C * kSB + j];
                const double g0 = fma(bn0, av[0], fma(bn1, av[1], fma(bn2, av[2], -bc)));
                const double g1 = fma(bn0, av[3], fma(bn1, av[4], fma(bn2, av[5], -bc)));
                const double g2 = fma(bn0, av[6], fma(bn1, av[7], fma(bn2, av[8], -bc)));
                if (separated(g0, g1, g2, tau)) continue;
                ++nex;
                const exact::tri ta{{av[0], av[1], av[2]}, {av[3], av[4], av[5]}, {av[6], av[7], av[8]}};
                const exact::tri tb{{bv[0], bv[kSB], bv[2 * kSB]}, {bv[3 * kSB], bv[4 * kSB], bv[5 * kSB]},
                                    {bv[6 * kSB], bv[7 * kSB], bv[8 * kSB]}};
                if (exact::tri_tri_hit(ta, tb)) {
                    atomicMin(a.objhit + o, i_loc * a.Bn + f0 + j);
                    done = true;  // later j of this row only give larger p
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && s + 2 < nsub) issue(s + 2);
    }
    if (nex) atomicAdd(a.nexact, nex);
}

}  // namespace

void run_intersects(const Ctx& cx, const ASel& sel, const Geom& B, uint8_t* hit, uint64_t* pair) {
    const cudaStream_t st = cx.stream;
    const uint64_t nobj = sel.obj1 - sel.obj0;
    const uint64_t ntiles = sel.tile1 - sel.tile0;
    const uint64_t n_items = ntiles * B.n_chunks;
    tdb_stats& S = *cx.stats;
    std::memset(&S, 0, sizeof S);
    for (uint64_t o = 0; o < nobj; ++o) {
        if (hit) hit[o] = 0;
        pair[o] = kNone;
    }
    if (nobj == 0 || n_items == 0) return;
    if (n_items > 0x7fffffffull) throw std::invalid_argument("intersects: too many work items for one launch");
    const Geom& A = *sel.A;
    unsigned long long *objhit = nullptr, *nex = nullptr;
    double* Bstats = nullptr;
    CK(cudaMallocAsync(&objhit, nobj * sizeof(unsigned long long), st));
    CK(cudaMallocAsync(&nex, sizeof(unsigned long long), st));
    CK(cudaMallocAsync(&Bstats, kObjStats * sizeof(double), st));
    CK(cudaMemsetAsync(objhit, 0xff, nobj * sizeof(unsigned long long), st));
    CK(cudaMemsetAsync(nex, 0, sizeof(unsigned long long), st));
    CK(cudaMemcpyAsync(Bstats, B.stats, kObjStats * sizeof(double), cudaMemcpyHostToDevice, st));
    cudaEvent_t e0, e1, e2;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventCreate(&e2));
    CK(cudaEventRecord(e0, st));
    hit_kernel<<<(unsigned)n_items, kTile, 0, st>>>(HitArgs{A.planes, A.n_pad, A.d_tiles, sel.tile0, sel.row_lo,
                                                            sel.row_hi, B.planes, B.n_pad, B.n, B.n_chunks,
                                                            sel.obj0, A.d_obj_stats, Bstats, objhit, nex});
    CK(cudaGetLastError());
    CK(cudaEventRecord(e1, st));
    std::vector<unsigned long long> hp(nobj);
    unsigned long long hn = 0;
    CK(cudaMemcpyAsync(hp.data(), objhit, nobj * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&hn, nex, sizeof hn, cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(e2, st));
    CK(cudaFreeAsync(objhit, st));
    CK(cudaFreeAsync(nex, st));
    CK(cudaFreeAsync(Bstats, st));
    CK(cudaStreamSynchronize(st));
    for (uint64_t o = 0; o < nobj; ++o) {
        pair[o] = hp[o];
        if (hit) hit[o] = hp[o] != kNone;
    }
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    S.ms_filter = ms;
    CK(cudaEventElapsedTime(&ms, e0, e2));
    S.ms_total = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
    uint64_t pairs = 0;
    for (uint64_t t = sel.tile0; t < sel.tile1; ++t) {
        const Tile& T = A.h_tiles[t];
        const uint64_t lo = std::max(T.row0, sel.row_lo), hi = std::min(T.row0 + T.count, sel.row_hi);
        if (hi > lo) pairs += (hi - lo) * B.n;
    }
    S.pairs = pairs;
    S.items = n_items;
    S.exact_pairs = hn;
    S.kernels = 1;
    S.rounds = 1;
}

}  // namespace tdb
