// Small calls (the serving path: one SQL literal, a handful of records, the
// shim's per-record distance_to_mesh) in ONE kernel launch each.
//
// The filter -> band -> verify pipeline (distance.cu, queries.cu) pays ~9
// launches and a host round trip per band round; below a few ten thousand
// pairs that overhead, not FP64 work, is the call. Here every pair runs the
// bit-exact reference composition directly (exact.cuh), so there is no band
// to certify:
//   * mesh x mesh distance: each thread evaluates exact::tri_tri on its pairs
//     and keeps the lexicographic (distance, pair) minimum with its witness;
//     CTAs reduce, and the last CTA to finish (ticket counter) reduces the CTA
//     results and writes the answer (kernels.cpp:359,368-376 tie rule);
//   * mesh x mesh intersects: exact::tri_tri_hit, atomicMin of the lowest hit
//     pair, pairs above the current lowest hit skipped (kernels.cpp:413-420);
//   * point / segment queries (<= kDirectQueries of them): one CTA per query,
//     threads over the faces, exact pt_tri / seg_tri (distance_to_mesh with
//     the mesh's has_degenerate_faces rule, kernels.cpp:347-378) or
//     seg_tri_hit (intersects_mesh, lowest hit face).
// Every evaluated pair also goes through the near-degenerate classifier
// (the same log as the exact pass). Results land in one small block copied
// back once.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <vector>

#include "exact.cuh"
#include "runtime.h"

namespace tdb {

namespace {

constexpr unsigned long long kNone = ~0ull;
constexpr int kDT = 128;  // threads per CTA

__device__ __forceinline__ exact::tri dtri(const double* P, uint64_t pad, uint64_t i) {
    double v[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) v[k] = __ldg(P + (uint64_t)(F_V + k) * pad + i);
    return exact::tri{{v[0], v[1], v[2]}, {v[3], v[4], v[5]}, {v[6], v[7], v[8]}};
}

__device__ __forceinline__ bool ddeg(const double* P, uint64_t pad, uint64_t i) {
    return __ldg(P + (uint64_t)F_DEG * pad + i) != 0.0;
}

// (distance bits, pair) lexicographic: a before b
__device__ __forceinline__ bool lex_lt(unsigned long long da, unsigned long long pa, unsigned long long db,
                                       unsigned long long pb) {
    return da < db || (da == db && pa < pb);
}

struct DirectDist {
    const double* Ap;
    uint64_t An_pad, row_lo, row_hi, obj_row0;
    const double* Bp;
    uint64_t Bn_pad, Bn;
    double* slots;                 // per CTA: d, p, witness[6]
    unsigned int* ticket;
    double* out;                   // d, p, witness[6]
    NearLog near;
};

// CTA-wide lexicographic min of (d, p) carrying a 6-double witness; thread 0
// returns it in r.
__device__ void cta_min(unsigned long long& d, unsigned long long& p, double* w) {
    __shared__ unsigned long long sd[kDT / 32], sp[kDT / 32];
    __shared__ double sw[kDT / 32][6];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long od = __shfl_xor_sync(0xffffffffu, d, o), op = __shfl_xor_sync(0xffffffffu, p, o);
        double ow[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) ow[k] = __shfl_xor_sync(0xffffffffu, w[k], o);
        if (lex_lt(od, op, d, p)) {
            d = od, p = op;
#pragma unroll
            for (int k = 0; k < 6; ++k) w[k] = ow[k];
        }
    }
    if (lane == 0) {
        sd[warp] = d, sp[warp] = p;
#pragma unroll
        for (int k = 0; k < 6; ++k) sw[warp][k] = w[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < kDT / 32; ++q)
            if (lex_lt(sd[q], sp[q], d, p)) {
                d = sd[q], p = sp[q];
                for (int k = 0; k < 6; ++k) w[k] = sw[q][k];
            }
    }
}

// The pair's six directed-edge seg_tri calls run on six lanes (a warp takes
// five pairs at a time); the group's first lane then scans them in the
// composition's order with the same first-strict-minimum rule, so the
// distance and witness are exact::tri_tri's bits.
constexpr int kGroups = 5;  // pairs per warp per step (6 lanes each)

__global__ void __launch_bounds__(kDT) direct_dist_kernel(DirectDist a) {
    const uint64_t rows = a.row_hi - a.row_lo, P = rows * a.Bn;
    unsigned long long bd = (unsigned long long)__double_as_longlong(__longlong_as_double(0x7ff0000000000000ll));
    unsigned long long bp = kNone;
    double w[6] = {0, 0, 0, 0, 0, 0};
    const int lane = threadIdx.x & 31, g = lane / 6, e = lane - 6 * g;  // g == 5: lanes 30, 31 idle
    const uint64_t warps = (uint64_t)gridDim.x * (kDT / 32);
    const uint64_t warp = (uint64_t)blockIdx.x * (kDT / 32) + (threadIdx.x >> 5);
    for (uint64_t k0 = warp * kGroups; k0 < P; k0 += warps * kGroups) {  // uniform per warp
        const uint64_t k = k0 + g;
        const bool mine = g < kGroups && k < P;
        const uint64_t i = a.row_lo + (mine ? k / a.Bn : 0), j = mine ? k % a.Bn : 0;
        const bool skip = !mine || ddeg(a.Ap, a.An_pad, i) || ddeg(a.Bp, a.Bn_pad, j);  // A17: degenerate pairs skipped
        exact::res c;
        c.d = __longlong_as_double(0x7ff0000000000000ll);
        c.a = c.b = exact::mk(0.0, 0.0, 0.0);
        exact::tri ta{}, tb{};
        if (!skip) {
            ta = dtri(a.Ap, a.An_pad, i), tb = dtri(a.Bp, a.Bn_pad, j);
            const exact::tri& src = e < 3 ? ta : tb;
            const exact::tri& dst = e < 3 ? tb : ta;
            const int q = e % 3;
            const exact::v3 p0 = q == 0 ? src.v0 : q == 1 ? src.v1 : src.v2;
            const exact::v3 p1 = q == 0 ? src.v1 : q == 1 ? src.v2 : src.v0;
            c = exact::seg_tri(p0, p1, dst);
            if (e >= 3) {  // edges of b against a: the witness is (point on a, point on b)
                const exact::v3 t = c.a;
                c.a = c.b, c.b = t;
            }
        }
        const int base = 6 * (g < kGroups ? g : 0);
        double cd[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) cd[q] = __shfl_sync(0xffffffffu, c.d, base + q);
        int win = -1;
        double best = __longlong_as_double(0x7ff0000000000000ll);
#pragma unroll
        for (int q = 0; q < 6; ++q)
            if (cd[q] < best) best = cd[q], win = q;
        const int src = base + (win < 0 ? 0 : win);
        double wv[6] = {c.a.x, c.a.y, c.a.z, c.b.x, c.b.y, c.b.z};
#pragma unroll
        for (int q = 0; q < 6; ++q) wv[q] = __shfl_sync(0xffffffffu, wv[q], src);
        if (e == 0 && !skip) {  // as exact::tri_tri: +inf and a zero witness when no candidate is below +inf
            const unsigned long long p = (i - a.obj_row0) * a.Bn + j;
            if (exact::near_degenerate_pair(ta, tb)) near_log(a.near, 0, p);
            const unsigned long long d = (unsigned long long)__double_as_longlong(best);
            if (lex_lt(d, p, bd, bp)) {
                bd = d, bp = p;
#pragma unroll
                for (int q = 0; q < 6; ++q) w[q] = win < 0 ? 0.0 : wv[q];
            }
        }
    }
    cta_min(bd, bp, w);
    if (gridDim.x == 1) {  // one CTA: its minimum is the answer
        if (threadIdx.x == 0) {
            a.out[0] = __longlong_as_double((long long)bd);
            a.out[1] = __longlong_as_double((long long)bp);
            for (int k = 0; k < 6; ++k) a.out[2 + k] = w[k];
        }
        return;
    }
    __shared__ bool last;
    if (threadIdx.x == 0) {
        double* s = a.slots + 8 * blockIdx.x;
        s[0] = __longlong_as_double((long long)bd);
        s[1] = __longlong_as_double((long long)bp);
        for (int k = 0; k < 6; ++k) s[2 + k] = w[k];
        __threadfence();
        last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    // the last CTA: reduce the CTA results (every slot is visible after the fence + ticket)
    __threadfence();
    if (threadIdx.x == 0) *a.ticket = 0;  // ready for the next call on this scratch
    bd = (unsigned long long)__double_as_longlong(__longlong_as_double(0x7ff0000000000000ll)), bp = kNone;
    for (int k = 0; k < 6; ++k) w[k] = 0.0;
    for (uint64_t c = threadIdx.x; c < gridDim.x; c += kDT) {
        const volatile double* s = a.slots + 8 * c;
        const unsigned long long d = (unsigned long long)__double_as_longlong(s[0]);
        const unsigned long long p = (unsigned long long)__double_as_longlong(s[1]);
        if (lex_lt(d, p, bd, bp)) {
            bd = d, bp = p;
            for (int k = 0; k < 6; ++k) w[k] = s[2 + k];
        }
    }
    cta_min(bd, bp, w);
    if (threadIdx.x == 0) {
        a.out[0] = __longlong_as_double((long long)bd);
        a.out[1] = __longlong_as_double((long long)bp);
        for (int k = 0; k < 6; ++k) a.out[2 + k] = w[k];
    }
}

struct DirectHit {
    const double* Ap;
    uint64_t An_pad, row_lo, row_hi, obj_row0;
    const double* Bp;
    uint64_t Bn_pad, Bn;
    unsigned long long* best;  // lowest hit pair
    NearLog near;
};

// pairs in ascending order per thread; a thread stops once the lowest hit so
// far is below its next pair (kernels.cpp:413-415)
__global__ void __launch_bounds__(kDT) direct_hit_kernel(DirectHit a) {
    const uint64_t rows = a.row_hi - a.row_lo, P = rows * a.Bn;
    for (uint64_t k = (uint64_t)blockIdx.x * kDT + threadIdx.x; k < P; k += (uint64_t)gridDim.x * kDT) {
        const uint64_t i = a.row_lo + k / a.Bn, j = k % a.Bn;
        const unsigned long long p = (i - a.obj_row0) * a.Bn + j;
        if (*(volatile unsigned long long*)a.best < p) return;
        if (ddeg(a.Ap, a.An_pad, i) || ddeg(a.Bp, a.Bn_pad, j)) continue;
        const exact::tri ta = dtri(a.Ap, a.An_pad, i), tb = dtri(a.Bp, a.Bn_pad, j);
        if (exact::near_degenerate_pair(ta, tb)) near_log(a.near, 0, p);
        if (exact::tri_tri_hit(ta, tb)) {
            atomicMin(a.best, p);
            return;
        }
    }
}

struct DirectQ {
    double q[kDirectQueries][6];
    int n, point, op, split;     // split: CTAs per query
    const double* Bp;
    uint64_t Bn_pad, Bn;
    const uint8_t* keep_deg;     // B's has_degenerate_faces == false
    unsigned long long* out;     // per query: d bits (or hit flag), face
    unsigned long long* slots;   // per (query, part): d bits, face
    unsigned int* tickets;       // per query (0 on entry; the reducing CTA resets it)
    NearLog near;
};

// One query per `split` CTAs, each over a contiguous range of the faces; the
// last CTA of a query (ticket) reduces the parts: lowest (distance, face) for
// distance_to_mesh, lowest hit face for intersects_mesh.
__global__ void __launch_bounds__(kDT) direct_q_kernel(DirectQ a) {
    const int qi = blockIdx.x / a.split, part = blockIdx.x - qi * a.split;
    const uint64_t len = (a.Bn + a.split - 1) / a.split;
    const uint64_t f0 = min(a.Bn, (uint64_t)part * len), f1 = min(a.Bn, f0 + len);
    const exact::v3 p0{a.q[qi][0], a.q[qi][1], a.q[qi][2]};
    const exact::v3 p1 = a.point ? p0 : exact::v3{a.q[qi][3], a.q[qi][4], a.q[qi][5]};
    const bool zero = !a.point && p0.x == p1.x && p0.y == p1.y && p0.z == p1.z;  // kernels.cpp:389: a point
    unsigned long long bd = (unsigned long long)__double_as_longlong(__longlong_as_double(0x7ff0000000000000ll));
    unsigned long long bf = kNone;
    double w[6] = {0, 0, 0, 0, 0, 0};
    if (a.op == TDB_OP_DISTANCE) {
        const bool skip = !a.keep_deg[0];
        for (uint64_t j = f0 + threadIdx.x; j < f1; j += kDT) {
            if (skip && ddeg(a.Bp, a.Bn_pad, j)) continue;  // kernels.cpp:350,357
            const exact::tri t = dtri(a.Bp, a.Bn_pad, j);
            const double d = (a.point || zero) ? exact::pt_tri(p0, t).d : exact::seg_tri(p0, p1, t).d;
            if ((a.point || zero) ? exact::near_area(t) : exact::near_degenerate_seg(p0, p1, t)) near_log(a.near, qi, j);
            const unsigned long long e = (unsigned long long)__double_as_longlong(d);
            if (e < bd) bd = e, bf = j;  // ascending faces per thread: strict < keeps the lowest
        }
        cta_min(bd, bf, w);
    } else {
        __shared__ unsigned long long lowest;
        if (threadIdx.x == 0) lowest = kNone;
        __syncthreads();
        for (uint64_t j = f0 + threadIdx.x; j < f1; j += kDT) {
            if (*(volatile unsigned long long*)&lowest < j) break;
            const exact::tri t = dtri(a.Bp, a.Bn_pad, j);
            if (exact::near_degenerate_seg(p0, p1, t)) near_log(a.near, qi, j);
            if (exact::seg_tri_hit(p0, p1, t)) {
                atomicMin(&lowest, (unsigned long long)j);
                break;
            }
        }
        __syncthreads();
        bf = lowest;
    }
    __shared__ bool last;
    if (threadIdx.x == 0) {
        a.slots[2 * blockIdx.x] = bd;
        a.slots[2 * blockIdx.x + 1] = bf;
        __threadfence();
        last = atomicAdd(a.tickets + qi, 1u) == (unsigned)a.split - 1;
    }
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence();
    a.tickets[qi] = 0;  // ready for the next call on this scratch
    // parts in face order: strict < keeps the lowest face on ties
    bd = (unsigned long long)__double_as_longlong(__longlong_as_double(0x7ff0000000000000ll)), bf = kNone;
    for (int c = 0; c < a.split; ++c) {
        const volatile unsigned long long* sl = a.slots + 2 * ((uint64_t)qi * a.split + c);
        const unsigned long long d = sl[0], f = sl[1];
        if (a.op == TDB_OP_DISTANCE ? (f != kNone && (bf == kNone || d < bd)) : f < bf) bd = d, bf = f;
    }
    a.out[2 * qi] = a.op == TDB_OP_DISTANCE ? bd : (unsigned long long)(bf != kNone);
    a.out[2 * qi + 1] = bf;
}

// Per (thread, device) scratch, kept across calls (a small call must not pay
// cudaMallocAsync / cudaFreeAsync): device block [near count | tickets (up to
// 62) | results | CTA slots | near entries] and a pinned host copy of its head.
struct Scratch {
    char* base = nullptr;
    unsigned long long* host = nullptr;  // pinned: near count, ticket, results
    unsigned long long* near_total = nullptr;
    size_t o_res = 0, o_nc = 0, o_ne = 0, o_slot = 0, o_tk = 0, head_bytes = 0;
};

struct DirectBuf {
    char* d = nullptr;
    size_t cap = 0;
    unsigned long long* h = nullptr;
    size_t hcap = 0;
    unsigned long long near_total = 0;  // the device near counter's value (never reset)
    ~DirectBuf() {  // thread exit; errors ignored (the context may be gone)
        if (d) cudaFree(d);
        if (h) cudaFreeHost(h);
    }
};

Scratch scratch(size_t res_bytes, size_t slot_bytes, cudaStream_t st) {
    thread_local std::vector<std::unique_ptr<DirectBuf>> per_device;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if ((int)per_device.size() <= dev) per_device.resize(dev + 1);
    if (!per_device[dev]) per_device[dev] = std::make_unique<DirectBuf>();
    DirectBuf& B = *per_device[dev];
    Scratch s;
    size_t off = 0;
    auto piece = [&](size_t b) {
        const size_t o = off;
        off = (off + std::max<size_t>(b, 8) + 255) & ~size_t(255);
        return o;
    };
    s.o_nc = 0;
    s.o_tk = 8;
    off = 256;
    s.o_res = piece(res_bytes);
    s.head_bytes = off;
    s.o_slot = piece(slot_bytes);
    s.o_ne = piece(2 * kNearLogCap * 8);
    if (B.cap < off) {
        if (B.d) CK(cudaFree(B.d));
        B.d = nullptr;
        B.cap = std::max(off, (size_t)1 << 17);
        CK(cudaMalloc(&B.d, B.cap));
        // the near counter and the tickets start at 0 once; afterwards the
        // tickets are reset by the CTA that reduces, and the counter only grows
        CK(cudaMemset(B.d, 0, 256));
        B.near_total = 0;
    }
    if (B.hcap < s.head_bytes) {
        if (B.h) CK(cudaFreeHost(B.h));
        B.h = nullptr;
        B.hcap = std::max(s.head_bytes, (size_t)4096);
        CK(cudaMallocHost(&B.h, B.hcap));
    }
    s.base = B.d;
    s.host = B.h;
    s.near_total = &B.near_total;
    (void)st;
    return s;
}

// Results back: the head (near count, results) in one copy to pinned memory;
// the near-degenerate entries only when there are any.
void finish(const Ctx& cx, Scratch& s, uint64_t pairs, int kernels, std::chrono::steady_clock::time_point t0) {
    const cudaStream_t st = cx.stream;
    CK(cudaMemcpyAsync(s.host, s.base, s.head_bytes, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    tdb_stats& S = *cx.stats;
    std::memset(&S, 0, sizeof S);
    // one launch: host wall time from the launch to the results (device
    // events would add two API calls to a call of a few ten microseconds)
    S.ms_total = S.ms_verify = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    S.pairs = S.pairs_evaluated = S.exact_pairs = S.candidates = pairs;
    S.kernels = kernels;
    S.rounds = 1;
    const unsigned long long total = s.host[s.o_nc / 8], nc = total - *s.near_total;
    *s.near_total = total;
    cx.near->count = nc;
    cx.near->entries.assign(2 * std::min<uint64_t>(nc, kNearLogCap), 0);
    if (nc) {
        CK(cudaMemcpyAsync(cx.near->entries.data(), s.base + s.o_ne, cx.near->entries.size() * 8,
                           cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    S.near_degenerate = nc;
}

uint64_t sel_rows(const ASel& sel) { return sel.row_hi - sel.row_lo; }

unsigned grid_for(uint64_t work, int sms) {
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((work + kDT - 1) / kDT, (uint64_t)sms * 8));
}

// direct_dist_kernel: one pair per 6 lanes, kGroups pairs per warp
unsigned grid_for_dist(uint64_t pairs, int sms) {
    const uint64_t per_cta = (uint64_t)kGroups * (kDT / 32);
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((pairs + per_cta - 1) / per_cta, (uint64_t)sms * 8));
}

}  // namespace

bool direct_eligible(const ASel& sel, const Geom& B, int op) {
    return sel.obj1 - sel.obj0 == 1 && sel_rows(sel) * B.n <= direct_pairs(op) && sel_rows(sel) * B.n > 0;
}

void run_distance_direct(const Ctx& cx, const ASel& sel, const Geom& B, double* dist, uint64_t* pair,
                         double* witness6) {
    const cudaStream_t st = cx.stream;
    const Geom& A = *sel.A;
    const uint64_t P = sel_rows(sel) * B.n;
    const unsigned grid = grid_for_dist(P, cx.sms);
    Scratch s = scratch(8 * sizeof(double), (size_t)grid * 8 * sizeof(double), st);
    const auto t0 = std::chrono::steady_clock::now();
    DirectDist a{A.planes, A.n_pad, sel.row_lo, sel.row_hi, A.h_off[sel.obj0], B.planes, B.n_pad, B.n,
                 (double*)(s.base + s.o_slot), (unsigned int*)(s.base + s.o_tk), (double*)(s.base + s.o_res),
                 NearLog{(unsigned long long*)(s.base + s.o_nc), (unsigned long long*)(s.base + s.o_ne), *s.near_total}};
    direct_dist_kernel<<<grid, kDT, 0, st>>>(a);
    CK(cudaGetLastError());
    finish(cx, s, P, 1, t0);
    const unsigned long long* r = s.host + s.o_res / 8;
    const unsigned long long p = r[1];
    *pair = p;
    if (p != kNone) std::memcpy(dist, &r[0], sizeof(double));
    else *dist = pos_inf_h();
    if (witness6) {
        if (p != kNone) std::memcpy(witness6, &r[2], 6 * sizeof(double));
        else std::fill(witness6, witness6 + 6, 0.0);
    }
}

void run_intersects_direct(const Ctx& cx, const ASel& sel, const Geom& B, uint8_t* hit, uint64_t* pair) {
    const cudaStream_t st = cx.stream;
    const Geom& A = *sel.A;
    const uint64_t P = sel_rows(sel) * B.n;
    Scratch s = scratch(8, 0, st);
    unsigned long long* best = (unsigned long long*)(s.base + s.o_res);
    CK(cudaMemsetAsync(best, 0xff, 8, st));
    const auto t0 = std::chrono::steady_clock::now();
    direct_hit_kernel<<<grid_for(P, cx.sms), kDT, 0, st>>>(
        DirectHit{A.planes, A.n_pad, sel.row_lo, sel.row_hi, A.h_off[sel.obj0], B.planes, B.n_pad, B.n, best,
                  NearLog{(unsigned long long*)(s.base + s.o_nc), (unsigned long long*)(s.base + s.o_ne), *s.near_total}});
    CK(cudaGetLastError());
    finish(cx, s, P, 1, t0);
    const unsigned long long p = s.host[s.o_res / 8];
    *pair = p;
    if (hit) *hit = p != kNone;
}

void run_queries_direct(const Ctx& cx, int op, const double* q, uint64_t n, int kind, const Geom& B, double* dist,
                        uint8_t* hit, uint64_t* face) {
    if (n == 0) return;
    const cudaStream_t st = cx.stream;
    DirectQ a{};
    const int width = kind == kQueryPoints ? 3 : 6;
    for (uint64_t i = 0; i < n; ++i)
        for (int k = 0; k < width; ++k) a.q[i][k] = q[width * i + k];
    a.n = (int)n;
    a.point = kind == kQueryPoints;
    a.op = op;
    a.Bp = B.planes;
    a.Bn_pad = B.n_pad;
    a.Bn = B.n;
    a.keep_deg = B.d_keep_deg;
    // enough CTAs that each thread sees a few faces (the exact composition per face is long)
    a.split = (int)std::max<uint64_t>(1, std::min<uint64_t>(32, (B.n + 2 * kDT - 1) / (2 * kDT)));
    Scratch s = scratch(2 * n * 8, 2 * 8 * n * (size_t)a.split, st);
    a.out = (unsigned long long*)(s.base + s.o_res);
    a.slots = (unsigned long long*)(s.base + s.o_slot);
    a.tickets = (unsigned int*)(s.base + s.o_tk);
    a.near = NearLog{(unsigned long long*)(s.base + s.o_nc), (unsigned long long*)(s.base + s.o_ne), *s.near_total};
    const auto t0 = std::chrono::steady_clock::now();
    direct_q_kernel<<<(unsigned)(n * a.split), kDT, 0, st>>>(a);
    CK(cudaGetLastError());
    finish(cx, s, n * B.n, 1, t0);
    const unsigned long long* r = s.host + s.o_res / 8;
    for (uint64_t i = 0; i < n; ++i) {
        const unsigned long long f = r[2 * i + 1];
        if (face) face[i] = f;
        if (op == TDB_OP_DISTANCE) {
            if (dist) {
                if (f != kNone) std::memcpy(&dist[i], &r[2 * i], sizeof(double));
                else dist[i] = pos_inf_h();
            }
        } else if (hit) {
            hit[i] = f != kNone;
        }
    }
}

}  // namespace tdb
