// Device geometry store: upload of caller-owned AoS triangle soups into
// per-face SoA planes in HBM, with per-object AABB headers and A-side tiles.
//
// Replaces the CPU mesh store for the hot path (store_types.hpp:14-32,
// geometry.hpp:81-98). The caller's array is exactly
// tindb::TriangleMesh::triangles.data() (72 B per face); it is copied once
// (H2D) into a staging buffer and transposed + enriched by prep_kernel.
#include <algorithm>
#include <cmath>
#include <vector>

#include "exact.cuh"
#include "runtime.h"

namespace tdb {

namespace {

__device__ __forceinline__ double pos_inf_h_d() { return __longlong_as_double(0x7ff0000000000000LL); }

// Order-preserving u64 encoding of doubles for atomicMin/atomicMax.
__device__ __forceinline__ unsigned long long ord(double d) {
    const unsigned long long u = (unsigned long long)__double_as_longlong(d);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double unord(unsigned long long u) {
    return __longlong_as_double((long long)((u >> 63) ? (u & 0x7fffffffffffffffull) : ~u));
}

__device__ __forceinline__ uint32_t object_of(const uint64_t* off, uint64_t n_obj, uint64_t face) {
    uint64_t lo = 0, hi = n_obj;  // off[lo] <= face < off[hi]
    while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (off[mid] <= face) lo = mid; else hi = mid;
    }
    return (uint32_t)lo;
}

// One thread per face: planes + per-object statistics (8 ordered u64 per
// object: lo xyz (min), hi xyz (max), max edge, max |coord|) + degenerate
// count.
__global__ void prep_kernel(const double* __restrict__ aos, uint64_t n, uint64_t n_pad,
                            const uint64_t* __restrict__ off, uint64_t n_obj,
                            double* __restrict__ planes, unsigned long long* __restrict__ stats,
                            unsigned long long* __restrict__ n_deg, float* __restrict__ fplanes, double ox,
                            double oy, double oz) {
    const uint64_t f = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = f < n;
    const uint64_t g = live ? f : (n ? n - 1 : 0);
    double v[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) v[k] = n ? aos[9 * g + k] : 0.0;

    exact::tri t{{v[0], v[1], v[2]}, {v[3], v[4], v[5]}, {v[6], v[7], v[8]}};
    const bool deg = exact::degenerate(t);

    double e[9], L[3], IL[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const int q = j == 2 ? 0 : j + 1;
        e[3 * j] = v[3 * q] - v[3 * j];
        e[3 * j + 1] = v[3 * q + 1] - v[3 * j + 1];
        e[3 * j + 2] = v[3 * q + 2] - v[3 * j + 2];
        L[j] = e[3 * j] * e[3 * j] + e[3 * j + 1] * e[3 * j + 1] + e[3 * j + 2] * e[3 * j + 2];
        IL[j] = L[j] > 0.0 ? 1.0 / L[j] : 0.0;
    }
    // e0 = V1 - V0 = E_0, e1 = V2 - V0 = -E_2
    const double a0 = e[0], a1 = e[1], a2 = e[2];
    const double b0 = -e[6], b1 = -e[7], b2 = -e[8];
    const double Nx = a1 * b2 - a2 * b1, Ny = a2 * b0 - a0 * b2, Nz = a0 * b1 - a1 * b0;
    const double N2 = Nx * Nx + Ny * Ny + Nz * Nz;
    double n3[3] = {0, 0, 0}, U[3] = {0, 0, 0}, W[3] = {0, 0, 0}, c = 0.0;
    // conditioning of the reference's solve against this face: its t / (u, v)
    // noise scales with K = |e0||e1|/|N|; +inf when N = 0
    const double kappa = N2 > 0.0 ? 8.0000001e-15 * sqrt((a0 * a0 + a1 * a1 + a2 * a2) * L[2] / N2)
                                  : __longlong_as_double(0x7ff0000000000000ll);
    if (!deg && N2 > 0.0) {
        const double inv = 1.0 / sqrt(N2), inv2 = 1.0 / N2;
        n3[0] = Nx * inv, n3[1] = Ny * inv, n3[2] = Nz * inv;
        c = n3[0] * v[0] + n3[1] * v[1] + n3[2] * v[2];
        // U = (e1 x N)/|N|^2, W = (N x e0)/|N|^2
        U[0] = (b1 * Nz - b2 * Ny) * inv2, U[1] = (b2 * Nx - b0 * Nz) * inv2, U[2] = (b0 * Ny - b1 * Nx) * inv2;
        W[0] = (Ny * a2 - Nz * a1) * inv2, W[1] = (Nz * a0 - Nx * a2) * inv2, W[2] = (Nx * a1 - Ny * a0) * inv2;
    } else {
        // degenerate: no vertex projects "inside" (NaN barycentrics fail every
        // inside test), so a face the queries evaluate anyway (its mesh's
        // has_degenerate_faces is false) gets only edge candidates, the
        // reference's fallback (kernels.cpp:127-134, 151-156, 262-316)
        const double nan = __longlong_as_double(0x7ff8000000000000ll);
        U[0] = U[1] = U[2] = W[0] = W[1] = W[2] = nan;
    }
    if (live) {
        double* p = planes + f;
#pragma unroll
        for (int k = 0; k < 9; ++k) p[(F_V + k) * n_pad] = v[k];
#pragma unroll
        for (int k = 0; k < 9; ++k) p[(F_E + k) * n_pad] = e[k];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            p[(F_L + k) * n_pad] = L[k];
            p[(F_IL + k) * n_pad] = IL[k];
            p[(F_N + k) * n_pad] = n3[k];
            p[(F_U + k) * n_pad] = U[k];
            p[(F_W + k) * n_pad] = W[k];
        }
        p[F_C * n_pad] = c;
        p[F_DEG * n_pad] = deg ? 1.0 : 0.0;
        p[F_K * n_pad] = kappa;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            p[(F_LO + k) * n_pad] = fmin(v[k], fmin(v[3 + k], v[6 + k]));
            p[(F_HI + k) * n_pad] = fmax(v[k], fmax(v[3 + k], v[6 + k]));
        }
        const double o3[3] = {ox, oy, oz};
#pragma unroll
        for (int k = 0; k < 3; ++k)  // vertex k as one float4 (x, y, z, 0) in plane k
            reinterpret_cast<float4*>(fplanes)[(uint64_t)k * n_pad + f] =
                make_float4(__double2float_rn(v[3 * k] - o3[0]), __double2float_rn(v[3 * k + 1] - o3[1]),
                            __double2float_rn(v[3 * k + 2] - o3[2]), 0.0f);
    }

    // ---- per-object statistics, warp-aggregated when the warp is one object
    const uint32_t obj = object_of(off, n_obj, g);
    double s[kObjStats];
    s[0] = fmin(v[0], fmin(v[3], v[6]));
    s[1] = fmin(v[1], fmin(v[4], v[7]));
    s[2] = fmin(v[2], fmin(v[5], v[8]));
    s[3] = fmax(v[0], fmax(v[3], v[6]));
    s[4] = fmax(v[1], fmax(v[4], v[7]));
    s[5] = fmax(v[2], fmax(v[5], v[8]));
    s[6] = sqrt(fmax(L[0], fmax(L[1], L[2])));
    s[7] = fmax(fmax(fmax(-s[0], s[3]), fmax(-s[1], s[4])), fmax(-s[2], s[5]));
    s[8] = deg ? 0.0 : kappa;
    unsigned long long* st = stats + (uint64_t)obj * kObjStats;
    const unsigned mask = __activemask();
    const uint32_t obj0 = __shfl_sync(mask, obj, 0);
    const bool uniform = __all_sync(mask, obj == obj0);
    if (uniform) {
#pragma unroll
        for (int k = 0; k < kObjStats; ++k) {
            double x = s[k];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double y = __shfl_xor_sync(mask, x, o);
                x = k < 3 ? fmin(x, y) : fmax(x, y);
            }
            s[k] = x;
        }
        if ((threadIdx.x & 31) == 0 && n) {
            for (int k = 0; k < 3; ++k) atomicMin(st + k, ord(s[k]));
            for (int k = 3; k < kObjStats; ++k) atomicMax(st + k, ord(s[k]));
        }
    } else if (n) {
        for (int k = 0; k < 3; ++k) atomicMin(st + k, ord(s[k]));
        for (int k = 3; k < kObjStats; ++k) atomicMax(st + k, ord(s[k]));
    }
    const unsigned dm = __ballot_sync(mask, live && deg);
    if ((threadIdx.x & 31) == 0 && dm) atomicAdd(n_deg, (unsigned long long)__popc(dm));
    // non-finite coordinates (the reference rejects them at construction,
    // geometry.hpp:16-18): counted in n_deg[1], the upload then fails
    bool bad = false;
#pragma unroll
    for (int k = 0; k < 9; ++k) bad |= !isfinite(v[k]);
    const unsigned bm = __ballot_sync(mask, live && bad);
    if ((threadIdx.x & 31) == 0 && bm) atomicAdd(n_deg + 1, (unsigned long long)__popc(bm));
}

__global__ void stats_init_kernel(unsigned long long* stats, uint64_t n_obj) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_obj * kObjStats) return;
    const int k = (int)(i % kObjStats);
    stats[i] = k < 3 ? ~0ull : 0ull;  // min slots start at +max, max slots at -max
}

__global__ void stats_final_kernel(const unsigned long long* __restrict__ in, double* __restrict__ out,
                                   uint64_t n) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = unord(in[i]);
}

// AABB of face ranges, one block per range: the A tiles (tiles != null) or
// uniform B chunks of `len` faces. Used by CULL mode item bounds.
__global__ void range_aabb_kernel(const double* __restrict__ planes, uint64_t n, uint64_t n_pad,
                                  const Tile* __restrict__ tiles, uint64_t len, double* __restrict__ out) {
    uint64_t c0, c1;
    if (tiles) {
        c0 = tiles[blockIdx.x].row0;
        c1 = c0 + tiles[blockIdx.x].count;
    } else {
        c0 = (uint64_t)blockIdx.x * len;
        c1 = min(n, c0 + len);
    }
    double lo[3] = {pos_inf(), pos_inf(), pos_inf()}, hi[3] = {-pos_inf(), -pos_inf(), -pos_inf()};
    for (uint64_t f = c0 + threadIdx.x; f < c1; f += blockDim.x)
        for (int k = 0; k < 9; ++k) {
            const double x = planes[(F_V + k) * n_pad + f];
            lo[k % 3] = fmin(lo[k % 3], x);
            hi[k % 3] = fmax(hi[k % 3], x);
        }
    __shared__ double red[6][32];
    for (int k = 0; k < 6; ++k) {
        double x = k < 3 ? lo[k] : hi[k - 3];
        for (int o = 16; o > 0; o >>= 1) {
            const double y = __shfl_xor_sync(0xffffffffu, x, o);
            x = k < 3 ? fmin(x, y) : fmax(x, y);
        }
        if ((threadIdx.x & 31) == 0) red[k][threadIdx.x >> 5] = x;
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        const int k = threadIdx.x;
        double x = red[k][0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) x = k < 3 ? fmin(x, red[k][w]) : fmax(x, red[k][w]);
        out[blockIdx.x * 6 + k] = x;
    }
}

}  // namespace

void geom_build(Geom* g, const double* host_tri9, uint64_t n, const uint64_t* host_off,
                uint64_t n_obj, cudaStream_t st, bool tri9_on_device) {
    g->n = n;
    g->n_obj = n_obj;
    g->n_pad = ((n + 1 + kPlanePad - 1) / kPlanePad) * kPlanePad;
    g->h_off.assign(host_off, host_off + n_obj + 1);

    // tiles: per object, kTile-face blocks (A role)
    g->h_tiles.clear();
    g->obj_tile0.assign(n_obj + 1, 0);
    for (uint64_t o = 0; o < n_obj; ++o) {
        g->obj_tile0[o] = g->h_tiles.size();
        for (uint64_t r = g->h_off[o]; r < g->h_off[o + 1]; r += kTile) {
            Tile t;
            t.row0 = r;
            t.obj_row0 = g->h_off[o];
            t.count = (uint32_t)std::min<uint64_t>(kTile, g->h_off[o + 1] - r);
            t.obj = (uint32_t)o;
            g->h_tiles.push_back(t);
        }
    }
    g->obj_tile0[n_obj] = g->h_tiles.size();
    g->n_chunks = (n + kChunk - 1) / kChunk;

    double* staging = nullptr;
    if (!tri9_on_device) CK(cudaMallocAsync(&staging, std::max<uint64_t>(1, 9 * n) * sizeof(double), st));
    CK(cudaMallocAsync(&g->planes, (size_t)NF * g->n_pad * sizeof(double), st));
    CK(cudaMallocAsync(&g->d_off, (n_obj + 1) * sizeof(uint64_t), st));
    CK(cudaMallocAsync(&g->d_tiles, std::max<size_t>(1, g->h_tiles.size()) * sizeof(Tile), st));
    CK(cudaMallocAsync(&g->d_obj_stats, std::max<uint64_t>(1, n_obj) * kObjStats * sizeof(double), st));
    CK(cudaMallocAsync(&g->d_tile_aabb, std::max<size_t>(1, g->h_tiles.size()) * 6 * sizeof(double), st));
    g->h_keep_deg.assign(std::max<uint64_t>(1, n_obj), 0);  // default: skip degenerate faces
    CK(cudaMallocAsync(&g->d_keep_deg, g->h_keep_deg.size(), st));
    CK(cudaMemsetAsync(g->d_keep_deg, 0, g->h_keep_deg.size(), st));
    unsigned long long* ustats = nullptr;
    unsigned long long* ndeg = nullptr;
    CK(cudaMallocAsync(&ustats, std::max<uint64_t>(1, n_obj) * kObjStats * sizeof(unsigned long long), st));
    CK(cudaMallocAsync(&ndeg, 2 * sizeof(unsigned long long), st));  // degenerate, non-finite
    CK(cudaMemsetAsync(ndeg, 0, 2 * sizeof(unsigned long long), st));
    CK(cudaMemsetAsync(g->planes, 0, (size_t)NF * g->n_pad * sizeof(double), st));
    CK(cudaMallocAsync(&g->fplanes, (size_t)3 * g->n_pad * sizeof(float4), st));
    CK(cudaMemsetAsync(g->fplanes, 0, (size_t)3 * g->n_pad * sizeof(float4), st));

    if (n && !tri9_on_device)
        h2d(staging, host_tri9, 9 * n * sizeof(double), st);
    const double* src = tri9_on_device ? host_tri9 : staging;
    CK(cudaMemcpyAsync(g->d_off, g->h_off.data(), (n_obj + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    if (!g->h_tiles.empty())
        CK(cudaMemcpyAsync(g->d_tiles, g->h_tiles.data(), g->h_tiles.size() * sizeof(Tile),
                           cudaMemcpyHostToDevice, st));
    if (n_obj) {
        const uint64_t m = n_obj * kObjStats;
        stats_init_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(ustats, n_obj);
        CK(cudaGetLastError());
    }
    if (n) {
        // FP32 frame origin: the first vertex of face 0 (one small read; no reduction needed)
        if (tri9_on_device) {
            CK(cudaMemcpyAsync(g->origin, src, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
        } else {
            std::copy(host_tri9, host_tri9 + 3, g->origin);
        }
        for (double& x : g->origin)
            if (!std::isfinite(x)) x = 0.0;  // rejected below (non-finite count)
        prep_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(src, n, g->n_pad, g->d_off, n_obj, g->planes, ustats,
                                                                ndeg, g->fplanes, g->origin[0], g->origin[1],
                                                                g->origin[2]);
        CK(cudaGetLastError());
        if (!g->h_tiles.empty()) {
            range_aabb_kernel<<<(unsigned)g->h_tiles.size(), 128, 0, st>>>(g->planes, n, g->n_pad, g->d_tiles, 0,
                                                                          g->d_tile_aabb);
            CK(cudaGetLastError());
        }
    }
    if (n_obj) {
        const uint64_t m = n_obj * kObjStats;
        stats_final_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(ustats, g->d_obj_stats, m);
        CK(cudaGetLastError());
    }
    unsigned long long nd2[2] = {0, 0};
    CK(cudaMemcpyAsync(nd2, ndeg, sizeof nd2, cudaMemcpyDeviceToHost, st));
    // overall AABB / scale (for the single-object case this is the object)
    std::vector<double> os(std::max<uint64_t>(1, n_obj) * kObjStats, 0.0);
    if (n_obj) CK(cudaMemcpyAsync(os.data(), g->d_obj_stats, n_obj * kObjStats * sizeof(double),
                                  cudaMemcpyDeviceToHost, st));
    if (staging) CK(cudaFreeAsync(staging, st));
    CK(cudaFreeAsync(ustats, st));
    CK(cudaFreeAsync(ndeg, st));
    CK(cudaStreamSynchronize(st));
    if (nd2[1])
        throw std::invalid_argument(std::to_string(nd2[1]) +
                                    " face(s) with non-finite coordinates (geometry.hpp:16-18 requires finite)");
    g->n_degenerate = nd2[0];
    double agg[kObjStats] = {pos_inf_h(), pos_inf_h(), pos_inf_h(), -pos_inf_h(), -pos_inf_h(), -pos_inf_h(), 0.0, 0.0, 0.0};
    for (uint64_t o = 0; o < n_obj; ++o) {
        if (g->h_off[o + 1] == g->h_off[o]) continue;
        const double* s = &os[o * kObjStats];
        for (int k = 0; k < 3; ++k) agg[k] = std::min(agg[k], s[k]);
        for (int k = 3; k < kObjStats; ++k) agg[k] = std::max(agg[k], s[k]);
    }
    std::copy(agg, agg + kObjStats, g->stats);
}

void chunk_aabbs(const Geom& g, uint64_t len, double* out, cudaStream_t st) {
    const uint64_t n_chunks = (g.n + len - 1) / len;
    if (!n_chunks) return;
    range_aabb_kernel<<<(unsigned)n_chunks, 256, 0, st>>>(g.planes, g.n, g.n_pad, nullptr, len, out);
    CK(cudaGetLastError());
}

// Stream-ordered frees back into the device pool (the store was allocated
// from it with cudaMallocAsync): a plain cudaFree hands the pages back to the
// driver, and the next large upload then waits for them to be mapped again.
// Every call that used the store has synchronized before it returns.
namespace {

// One CTA (kFB threads, one per face) per feature block: bitwise-distinct
// vertices and unordered-vertex-pair edges of the block's non-degenerate
// faces, packed as [faces | vertices | edges] (tdb_internal.h). A vertex or
// edge is represented by its first occurrence in face order.
__global__ void __launch_bounds__(kFB) fblock_kernel(const double* __restrict__ planes, uint64_t n, uint64_t n_pad,
                                                     double* __restrict__ out, uint4* __restrict__ hdr,
                                                     double4* __restrict__ sph, unsigned* __restrict__ max_used) {
    constexpr int R = 3 * kFB;  // vertex / edge references of the block
    __shared__ unsigned long long vx[R], vy[R], vz[R];
    __shared__ int rep[R];
    __shared__ unsigned ekey[R];
    __shared__ int live_s[kFB];
    __shared__ int scan[3][kFB + 1];
    const int t = threadIdx.x;
    const uint64_t blk = blockIdx.x, f = blk * kFB + t;
    const bool live = f < n && planes[(uint64_t)F_DEG * n_pad + f] == 0.0;
    live_s[t] = live;
    double v[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) v[k] = f < n ? planes[(uint64_t)(F_V + k) * n_pad + f] : 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        vx[3 * t + k] = (unsigned long long)__double_as_longlong(v[3 * k]);
        vy[3 * t + k] = (unsigned long long)__double_as_longlong(v[3 * k + 1]);
        vz[3 * t + k] = (unsigned long long)__double_as_longlong(v[3 * k + 2]);
    }
    __syncthreads();
    int uv[3], ue[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int r = 3 * t + k;
        int rr = r;
        if (live)
            for (int q = 0; q < r; ++q)
                if (live_s[q / 3] && vx[q] == vx[r] && vy[q] == vy[r] && vz[q] == vz[r]) {
                    rr = q;
                    break;
                }
        rep[r] = rr;
        uv[k] = live && rr == r;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const unsigned a = (unsigned)rep[3 * t + k], b = (unsigned)rep[3 * t + (k == 2 ? 0 : k + 1)];
        ekey[3 * t + k] = min(a, b) << 16 | max(a, b);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int r = 3 * t + k;
        bool first = live;
        if (live)
            for (int q = 0; q < r; ++q)
                if (live_s[q / 3] && ekey[q] == ekey[r]) {
                    first = false;
                    break;
                }
        ue[k] = first;
    }
    // exclusive scans of (faces, vertices, edges) over the block's threads
    if (t == 0) scan[0][0] = scan[1][0] = scan[2][0] = 0;
    __syncthreads();
    if (t == 0) {
        for (int q = 0; q < kFB; ++q) scan[0][q + 1] = scan[0][q] + live_s[q];
    }
    scan[1][t + 1] = uv[0] + uv[1] + uv[2];
    scan[2][t + 1] = ue[0] + ue[1] + ue[2];
    __syncthreads();
    if (t == 0) {
        for (int q = 0; q < kFB; ++q) {
            scan[1][q + 1] += scan[1][q];
            scan[2][q + 1] += scan[2][q];
        }
    }
    __syncthreads();
    const int NF = scan[0][kFB], NV = scan[1][kFB], NE = scan[2][kFB];

    double* base = out + blk * (uint64_t)kFBCap;
    if (live) {
        double* fp = base + (uint64_t)kFP * scan[0][t];
        double* fv = base + (uint64_t)kFP * NF + (uint64_t)kFV * scan[0][t];
#pragma unroll
        for (int k = 0; k < 9; ++k) fv[FV_V + k] = v[k];
        fv[FV_IDX] = __longlong_as_double((long long)f);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            fp[FP_N + k] = planes[(uint64_t)(F_N + k) * n_pad + f];
            fp[FP_U + k] = planes[(uint64_t)(F_U + k) * n_pad + f];
            fp[FP_W + k] = planes[(uint64_t)(F_W + k) * n_pad + f];
        }
        fp[9] = 0.0;
        int vs = scan[1][t], es = scan[2][t];
        double* vr = base + (uint64_t)(kFP + kFV) * NF;
        double* er = vr + (uint64_t)kVR * NV;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            if (uv[k]) {
                double* p = vr + (uint64_t)kVR * vs++;
                p[0] = v[3 * k], p[1] = v[3 * k + 1], p[2] = v[3 * k + 2], p[3] = 0.0;
            }
            if (ue[k]) {
                double* p = er + (uint64_t)kER * es++;
                p[ER_P] = v[3 * k], p[ER_P + 1] = v[3 * k + 1], p[ER_P + 2] = v[3 * k + 2];
#pragma unroll
                for (int c = 0; c < 3; ++c) p[ER_E + c] = planes[(uint64_t)(F_E + 3 * k + c) * n_pad + f];
                p[ER_L] = planes[(uint64_t)(F_L + k) * n_pad + f];
                p[ER_IL] = planes[(uint64_t)(F_IL + k) * n_pad + f];
            }
        }
    }
    // bounding sphere of the block's live vertices (the filter's "can any
    // face of this block straddle the plane" test): box centre, max distance
    // rounded up
    {
        __shared__ double red[6][kFB];
        double lo[3] = {pos_inf_h_d(), pos_inf_h_d(), pos_inf_h_d()}, hi[3] = {-lo[0], -lo[0], -lo[0]};
        if (live)
            for (int k = 0; k < 9; ++k) lo[k % 3] = fmin(lo[k % 3], v[k]), hi[k % 3] = fmax(hi[k % 3], v[k]);
        for (int c = 0; c < 3; ++c) red[c][t] = lo[c], red[3 + c][t] = hi[c];
        __syncthreads();
        for (int w = kFB / 2; w > 0; w >>= 1) {
            if (t < w)
                for (int c = 0; c < 3; ++c)
                    red[c][t] = fmin(red[c][t], red[c][t + w]), red[3 + c][t] = fmax(red[3 + c][t], red[3 + c][t + w]);
            __syncthreads();
        }
        const double cx = 0.5 * (red[0][0] + red[3][0]), cy = 0.5 * (red[1][0] + red[4][0]),
                     cz = 0.5 * (red[2][0] + red[5][0]);
        __syncthreads();
        double r = 0.0;
        if (live)
            for (int k = 0; k < 3; ++k) {
                const double dx = v[3 * k] - cx, dy = v[3 * k + 1] - cy, dz = v[3 * k + 2] - cz;
                r = fmax(r, sqrt(dx * dx + dy * dy + dz * dz));
            }
        red[0][t] = r;
        __syncthreads();
        for (int w = kFB / 2; w > 0; w >>= 1) {
            if (t < w) red[0][t] = fmax(red[0][t], red[0][t + w]);
            __syncthreads();
        }
        if (t == 0) sph[blk] = make_double4(cx, cy, cz, red[0][0] * (1.0 + 1e-12));  // NaN / +inf when no live face
    }
    if (t == 0) {
        const unsigned used = (unsigned)((kFP + kFV) * NF + kVR * NV + kER * NE);
        hdr[blk] = make_uint4((unsigned)NF, (unsigned)NV, (unsigned)NE, used);
        atomicMax(max_used, used);
        atomicMax(max_used + 1, (unsigned)((kFP + kFV) * NF + kVR * NV));  // filter_kernel (FULL)
        atomicMax(max_used + 2, (unsigned)(kER * NE));             // edge_kernel
        atomicMax(max_used + 3, (unsigned)((kFP + kFV) * NF));     // vertex_kernel
    }
}

}  // namespace

void geom_edge_tiles(const Geom& g, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(*g.fmu);
    if (g.atiles_built) return;
    geom_super_tiles(g, st);  // the super-tiles' distinct edges and vertices (atiles.cu)
    CK(cudaStreamSynchronize(st));
    g.atiles_built = true;
}

namespace {
// Bounding sphere of each group of `group` consecutive faces (all faces,
// degenerate ones included): box centre, max vertex distance rounded up.
__global__ void group_sphere_kernel(const double* __restrict__ planes, uint64_t n, uint64_t n_pad, int group,
                                    double4* __restrict__ out) {
    __shared__ double red[6][128];
    const int t = threadIdx.x;
    const uint64_t g0 = (uint64_t)blockIdx.x * group;
    double lo[3] = {pos_inf_h_d(), pos_inf_h_d(), pos_inf_h_d()}, hi[3] = {-lo[0], -lo[0], -lo[0]};
    for (int i = t; i < group; i += blockDim.x) {
        const uint64_t f = g0 + i;
        if (f >= n) break;
        for (int k = 0; k < 9; ++k) {
            const double x = planes[(uint64_t)(F_V + k) * n_pad + f];
            lo[k % 3] = fmin(lo[k % 3], x), hi[k % 3] = fmax(hi[k % 3], x);
        }
    }
    for (int c = 0; c < 3; ++c) red[c][t] = lo[c], red[3 + c][t] = hi[c];
    __syncthreads();
    for (int w = 64; w > 0; w >>= 1) {
        if (t < w)
            for (int c = 0; c < 3; ++c)
                red[c][t] = fmin(red[c][t], red[c][t + w]), red[3 + c][t] = fmax(red[3 + c][t], red[3 + c][t + w]);
        __syncthreads();
    }
    const double cx = 0.5 * (red[0][0] + red[3][0]), cy = 0.5 * (red[1][0] + red[4][0]), cz = 0.5 * (red[2][0] + red[5][0]);
    __syncthreads();
    double r = 0.0;
    for (int i = t; i < group; i += blockDim.x) {
        const uint64_t f = g0 + i;
        if (f >= n) break;
        for (int k = 0; k < 3; ++k) {
            const double dx = planes[(uint64_t)(F_V + 3 * k) * n_pad + f] - cx;
            const double dy = planes[(uint64_t)(F_V + 3 * k + 1) * n_pad + f] - cy;
            const double dz = planes[(uint64_t)(F_V + 3 * k + 2) * n_pad + f] - cz;
            r = fmax(r, sqrt(dx * dx + dy * dy + dz * dz));
        }
    }
    red[0][t] = r;
    __syncthreads();
    for (int w = 64; w > 0; w >>= 1) {
        if (t < w) red[0][t] = fmax(red[0][t], red[0][t + w]);
        __syncthreads();
    }
    if (t == 0) out[blockIdx.x] = make_double4(cx, cy, cz, red[0][0] * (1.0 + 1e-12));
}
}  // namespace

void geom_hit_spheres(const Geom& g, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(*g.fmu);
    if (g.d_hsph || g.n == 0) return;
    const uint64_t ng = (g.n + kHitGroup - 1) / kHitGroup;
    double4* out = nullptr;
    CK(cudaMallocAsync(&out, ng * sizeof(double4), st));
    group_sphere_kernel<<<(unsigned)ng, 128, 0, st>>>(g.planes, g.n, g.n_pad, kHitGroup, out);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    g.d_hsph = out;
}

void geom_bedges(const Geom& g, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(*g.fmu);
    if (!g.h_bseoff.empty()) return;
    geom_super_bedges(g, st);
    CK(cudaStreamSynchronize(st));
}

void geom_feature_blocks(const Geom& g, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(*g.fmu);
    if (g.fblocks || g.n == 0) return;
    const uint64_t nb = (g.n + kFB - 1) / kFB;
    double* blocks = nullptr;
    uint4* hdr = nullptr;
    unsigned* mx = nullptr;
    CK(cudaMallocAsync(&blocks, nb * (uint64_t)kFBCap * sizeof(double), st));
    CK(cudaMallocAsync(&hdr, nb * sizeof(uint4), st));
    CK(cudaMallocAsync(&mx, 4 * sizeof(unsigned), st));
    CK(cudaMemsetAsync(mx, 0, 4 * sizeof(unsigned), st));
    double4* sph = nullptr;
    CK(cudaMallocAsync(&sph, nb * sizeof(double4), st));
    fblock_kernel<<<(unsigned)nb, kFB, 0, st>>>(g.planes, g.n, g.n_pad, blocks, hdr, sph, mx);
    CK(cudaGetLastError());
    unsigned used[4] = {0, 0, 0, 0};
    CK(cudaMemcpyAsync(used, mx, sizeof used, cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(mx, st));
    CK(cudaStreamSynchronize(st));
    g.fblocks = blocks;
    g.d_fhdr = hdr;
    g.d_fsph = sph;
    g.n_fblocks = nb;
    g.fblock_max = used[0];
    g.fblock_max_pfv = used[1];
    g.fblock_max_e = used[2];
    g.fblock_max_f = used[3];
}

void geom_release(Geom* g, cudaStream_t st) {
    if (!g) return;
    cudaFreeAsync(g->fblocks, st);
    cudaFreeAsync(g->d_fhdr, st);
    cudaFreeAsync(g->d_fsph, st);
    g->d_fsph = nullptr;
    cudaFreeAsync(g->aedges, st);
    cudaFreeAsync(g->averts, st);
    g->aedges = g->averts = nullptr;
    cudaFreeAsync(g->bedges, st);
    cudaFreeAsync(g->d_bseoff, st);
    cudaFreeAsync(g->d_hsph, st);
    g->d_hsph = nullptr;
    g->bedges = nullptr;
    g->d_bseoff = nullptr;
    g->h_bseoff.clear();
    g->h_tile_eoff.clear();
    g->h_tile_voff.clear();
    g->h_tile_st.clear();
    g->atiles_built = false;
    g->fblocks = nullptr;
    g->d_fhdr = nullptr;
    cudaFreeAsync(g->planes, st);
    cudaFreeAsync(g->d_off, st);
    cudaFreeAsync(g->d_tiles, st);
    cudaFreeAsync(g->d_obj_stats, st);
    cudaFreeAsync(g->d_tile_aabb, st);
    cudaFreeAsync(g->fplanes, st);
    cudaFreeAsync(g->d_keep_deg, st);
    g->planes = nullptr;
    g->fplanes = nullptr;
    g->d_keep_deg = nullptr;
}

}  // namespace tdb
