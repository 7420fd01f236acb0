// ST_3DVolume (the paper's third operator): signed divergence-theorem volume
// of a mesh, bit-identical to the reference mesh_volume (kernels.cpp:23-46).
//
// The reference fixes the summation tree so every backend agrees: faces are
// cut into chunks of cfg.chunk_size (executor.hpp:20-44, default 4096), each
// chunk is summed sequentially in face order, and the chunk partials are
// combined by the pairwise tree of pairwise_tree_sum (kernels.cpp:11-21).
// Here all face terms are computed in parallel first; then one thread sums
// one chunk in order with round-to-nearest intrinsics (no contraction), and
// one thread walks the tree — the same operations in the same order, so the
// same bits.
//
// Volume policy: permissive (the reference default) — the signed sum is
// returned for any mesh; watertightness (validate_closed, closure.cpp) is not
// evaluated on the device.
#include <algorithm>
#include <cstring>
#include <vector>

#include "exact.cuh"
#include "runtime.h"

namespace tdb {

namespace {

// kernels.cpp:23-25: dot(v0, (v1-v0) x (v2-v0)) / 6
__device__ __forceinline__ double face_term(const double* P, uint64_t pad, uint64_t i) {
    const exact::v3 v0{P[(F_V + 0) * pad + i], P[(F_V + 1) * pad + i], P[(F_V + 2) * pad + i]};
    const exact::v3 v1{P[(F_V + 3) * pad + i], P[(F_V + 4) * pad + i], P[(F_V + 5) * pad + i]};
    const exact::v3 v2{P[(F_V + 6) * pad + i], P[(F_V + 7) * pad + i], P[(F_V + 8) * pad + i]};
    const exact::v3 n = exact::cross(exact::sub(v1, v0), exact::sub(v2, v0));
    return __ddiv_rn(exact::dot(v0, n), 6.0);
}

// Phase 1: every face term, one thread per face (coalesced plane reads).
__global__ void terms_kernel(const double* __restrict__ P, uint64_t pad, uint64_t n, double* __restrict__ terms) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) terms[i] = face_term(P, pad, i);
}

// Phase 2: each chunk summed in face order (the reference's sequential
// accumulation) by one warp: the lanes load 32 consecutive terms coalesced
// (the next 32 prefetched), and every lane adds them in order from shuffles,
// so all lanes hold the same sum; lane 0 stores it.
__device__ __forceinline__ double ordered_sum_warp(const double* __restrict__ t, uint64_t b, uint64_t e) {
    const int lane = threadIdx.x & 31;
    double acc = 0.0;
    double next = b + lane < e ? __ldg(t + b + lane) : 0.0;
    for (uint64_t base = b; base < e; base += 32) {
        const double cur = next;
        if (base + 32 < e) next = base + 32 + lane < e ? __ldg(t + base + 32 + lane) : 0.0;
        const int cnt = (int)min((uint64_t)32, e - base);
        for (int k = 0; k < cnt; ++k) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, cur, k));
    }
    return acc;
}

__global__ void chunk_sums_kernel(const double* __restrict__ terms, uint64_t n, uint64_t chunk, uint64_t n_chunks,
                                  double* __restrict__ leaves) {
    const uint64_t k = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // one warp per chunk
    if (k >= n_chunks) return;
    const uint64_t b = k * chunk, e = min(n, b + chunk);
    const double v = ordered_sum_warp(terms, b, e);
    if ((threadIdx.x & 31) == 0) leaves[k] = v;
}

// kernels.cpp:11-21 pairwise_tree_sum, in place
__global__ void tree_sum_kernel(double* leaves, uint64_t size, double* out) {
    if (size == 0) {
        *out = 0.0;
        return;
    }
    while (size > 1) {
        uint64_t w = 0, i = 0;
        for (; i + 1 < size; i += 2) leaves[w++] = __dadd_rn(leaves[i], leaves[i + 1]);
        if (i < size) leaves[w++] = leaves[i];
        size = w;
    }
    *out = leaves[0];
}

// per-object leaves: leaf k covers faces [lb[k], le[k])
__global__ void leaf_sums_kernel(const double* __restrict__ terms, const uint64_t* __restrict__ lb,
                                 const uint64_t* __restrict__ le, uint64_t n_leaves, double* __restrict__ leaves) {
    const uint64_t k = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // one warp per leaf
    if (k >= n_leaves) return;
    const double v = ordered_sum_warp(terms, lb[k], le[k]);
    if ((threadIdx.x & 31) == 0) leaves[k] = v;
}

// pairwise_tree_sum per object over its leaves [l0[o], l0[o+1])
__global__ void object_trees_kernel(double* leaves, const uint64_t* __restrict__ l0, uint64_t n_obj,
                                    double* __restrict__ out) {
    const uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= n_obj) return;
    double* L = leaves + l0[o];
    uint64_t size = l0[o + 1] - l0[o];
    if (size == 0) {
        out[o] = 0.0;
        return;
    }
    while (size > 1) {
        uint64_t w = 0, i = 0;
        for (; i + 1 < size; i += 2) L[w++] = __dadd_rn(L[i], L[i + 1]);
        if (i < size) L[w++] = L[i];
        size = w;
    }
    out[o] = L[0];
}

}  // namespace

// mesh_volume of every object of a table (run_batch(Volume, ...) over a mesh
// column, batch.cpp:23-29): each object gets its own chunk tree, exactly as
// eval_volume calls mesh_volume per record with the caller's chunk_size.
void run_volume_table(const Ctx& cx, const Geom& g, uint64_t chunk, double* out) {
    const cudaStream_t st = cx.stream;
    if (chunk == 0) chunk = 4096;
    std::vector<uint64_t> lb, le, l0(g.n_obj + 1, 0);
    for (uint64_t o = 0; o < g.n_obj; ++o) {
        l0[o] = lb.size();
        for (uint64_t b = g.h_off[o]; b < g.h_off[o + 1]; b += chunk) {
            lb.push_back(b);
            le.push_back(std::min(g.h_off[o + 1], b + chunk));
        }
    }
    l0[g.n_obj] = lb.size();
    const uint64_t nl = lb.size();
    uint64_t *d_lb = nullptr, *d_le = nullptr, *d_l0 = nullptr;
    double *leaves = nullptr, *d_out = nullptr;
    CK(cudaMallocAsync(&d_lb, std::max<uint64_t>(1, nl) * sizeof(uint64_t), st));
    CK(cudaMallocAsync(&d_le, std::max<uint64_t>(1, nl) * sizeof(uint64_t), st));
    CK(cudaMallocAsync(&d_l0, (g.n_obj + 1) * sizeof(uint64_t), st));
    CK(cudaMallocAsync(&leaves, std::max<uint64_t>(1, nl) * sizeof(double), st));
    CK(cudaMallocAsync(&d_out, std::max<uint64_t>(1, g.n_obj) * sizeof(double), st));
    h2d(d_lb, lb.data(), nl * sizeof(uint64_t), st);
    h2d(d_le, le.data(), nl * sizeof(uint64_t), st);
    h2d(d_l0, l0.data(), (g.n_obj + 1) * sizeof(uint64_t), st);
    double* terms = nullptr;
    CK(cudaMallocAsync(&terms, std::max<uint64_t>(1, g.n) * sizeof(double), st));
    if (g.n) {
        terms_kernel<<<(unsigned)((g.n + 255) / 256), 256, 0, st>>>(g.planes, g.n_pad, g.n, terms);
        CK(cudaGetLastError());
    }
    if (nl) {
        leaf_sums_kernel<<<(unsigned)((nl * 32 + 127) / 128), 128, 0, st>>>(terms, d_lb, d_le, nl, leaves);
        CK(cudaGetLastError());
    }
    if (g.n_obj) {
        object_trees_kernel<<<(unsigned)((g.n_obj + 127) / 128), 128, 0, st>>>(leaves, d_l0, g.n_obj, d_out);
        CK(cudaGetLastError());
        d2h(out, d_out, g.n_obj * sizeof(double), st);
    }
    CK(cudaFreeAsync(d_lb, st));
    CK(cudaFreeAsync(d_le, st));
    CK(cudaFreeAsync(d_l0, st));
    CK(cudaFreeAsync(leaves, st));
    CK(cudaFreeAsync(terms, st));
    CK(cudaFreeAsync(d_out, st));
    CK(cudaStreamSynchronize(st));
    std::memset(cx.stats, 0, sizeof *cx.stats);
    cx.stats->kernels = (g.n ? 1 : 0) + (nl ? 1 : 0) + (g.n_obj ? 1 : 0);
}

double run_volume(const Ctx& cx, const Geom& g, uint64_t chunk) {
    const cudaStream_t st = cx.stream;
    if (chunk == 0) chunk = 4096;  // ExecutorConfig::chunk_size default (executor.hpp:23)
    const uint64_t n_chunks = (g.n + chunk - 1) / chunk;
    double *leaves = nullptr, *out = nullptr, *terms = nullptr;
    CK(cudaMallocAsync(&leaves, std::max<uint64_t>(1, n_chunks) * sizeof(double), st));
    CK(cudaMallocAsync(&out, sizeof(double), st));
    CK(cudaMallocAsync(&terms, std::max<uint64_t>(1, g.n) * sizeof(double), st));
    if (n_chunks) {
        terms_kernel<<<(unsigned)((g.n + 255) / 256), 256, 0, st>>>(g.planes, g.n_pad, g.n, terms);
        CK(cudaGetLastError());
        chunk_sums_kernel<<<(unsigned)((n_chunks * 32 + 127) / 128), 128, 0, st>>>(terms, g.n, chunk, n_chunks, leaves);
        CK(cudaGetLastError());
    }
    tree_sum_kernel<<<1, 1, 0, st>>>(leaves, n_chunks, out);
    CK(cudaGetLastError());
    double v = 0.0;
    CK(cudaMemcpyAsync(&v, out, sizeof v, cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(leaves, st));
    CK(cudaFreeAsync(out, st));
    CK(cudaFreeAsync(terms, st));
    CK(cudaStreamSynchronize(st));
    std::memset(cx.stats, 0, sizeof *cx.stats);
    cx.stats->kernels = n_chunks ? 3 : 1;
    return v;
}

}  // namespace tdb
