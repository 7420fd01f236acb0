// Aligned triangle-pair batches (golden vectors / parity) and the FP64
// issue-rate microbenchmark used as the roofline denominator.
#include <cstring>

#include "exact.cuh"
#include "runtime.h"

namespace tdb {

namespace {

__device__ __forceinline__ exact::tri tri_at(const double* t9, uint64_t k) {
    const double* v = t9 + 9 * k;
    return exact::tri{{v[0], v[1], v[2]}, {v[3], v[4], v[5]}, {v[6], v[7], v[8]}};
}

__global__ void pairs_kernel(const double* __restrict__ a9, const double* __restrict__ b9, uint64_t n,
                             double* __restrict__ dist, uint8_t* __restrict__ hit) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const exact::tri a = tri_at(a9, k), b = tri_at(b9, k);
        if (dist) dist[k] = exact::tri_tri(a, b).d;
        if (hit) hit[k] = exact::tri_tri_hit(a, b) ? 1 : 0;
    }
}

// FP64 filter value d~^2 for aligned pairs (tests the filter's accuracy).

__global__ void filter_pairs_kernel(const double* __restrict__ pa, const double* __restrict__ pb, uint64_t n,
                                    double* __restrict__ d2) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (uint64_t)gridDim.x * blockDim.x) {
        AFace A;
        load_aface(A, FaceRef{pa + NF * k, 1});
        const bool deg = pa[NF * k + F_DEG] != 0.0 || pb[NF * k + F_DEG] != 0.0;
        d2[k] = deg ? pos_inf() : pair_d2(A, FaceRef{pb + NF * k, 1}, pa + NF * k, 1);
    }
}

// FULL mode's candidate set per pair: the FP64 vertex/face candidates and
// piercing test, the nine edge/edge candidates in FP32 relative to o
// (edge32_kernel's arithmetic, fast_pair.cuh edge_pair32).
__global__ void filter_pairs_f32_kernel(const double* __restrict__ pa, const double* __restrict__ pb, uint64_t n,
                                        double ox, double oy, double oz, double* __restrict__ d2) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const double* fa = pa + NF * k;
        const double* fb = pb + NF * k;
        AFace A;
        load_aface(A, FaceRef{fa, 1});
        if (fa[F_DEG] != 0.0 || fb[F_DEG] != 0.0) {
            d2[k] = pos_inf();
            continue;
        }
        const double v = pair_d2<FaceRef, false>(A, FaceRef{fb, 1}, fa, 1);
        float best = __int_as_float(0x7f800000);
        float q[3][8];
        for (int i = 0; i < 3; ++i) {
            const float qi[8] = {(float)(fa[F_V + 3 * i] - ox), (float)(fa[F_V + 3 * i + 1] - oy),
                                 (float)(fa[F_V + 3 * i + 2] - oz), (float)fa[F_E + 3 * i], (float)fa[F_E + 3 * i + 1],
                                 (float)fa[F_E + 3 * i + 2], (float)fa[F_L + i], (float)fa[F_IL + i]};
            for (int f = 0; f < 8; ++f) q[i][f] = qi[f];
        }
        // the packed form (edge_pair32x2) on A edges {0, 1} and {2, 2}: any
        // bit difference from the scalar one is reported as NaN
        AEdge32x2 A2[2];
        for (int h = 0; h < 2; ++h) {
            const float* x = q[2 * h];
            const float* y = q[h == 0 ? 1 : 2];
            for (int c = 0; c < 3; ++c)
                A2[h].q[c] = pk2f(x[c], y[c]), A2[h].e[c] = pk2f(x[3 + c], y[3 + c]),
                A2[h].ne[c] = pk2f(-x[3 + c], -y[3 + c]);
            A2[h].L = pk2f(x[6], y[6]);
            A2[h].il[0] = x[7], A2[h].il[1] = y[7];
        }
        bool same = true;
        for (int j = 0; j < 3; ++j) {
            const float4 p0 = make_float4((float)(fb[F_V + 3 * j] - ox), (float)(fb[F_V + 3 * j + 1] - oy),
                                          (float)(fb[F_V + 3 * j + 2] - oz), (float)fb[F_E + 3 * j]);
            const float4 p1 = make_float4((float)fb[F_E + 3 * j + 1], (float)fb[F_E + 3 * j + 2],
                                          (float)fb[F_L + j], (float)fb[F_IL + j]);
            float e[3];
            for (int i = 0; i < 3; ++i) {
                e[i] = edge_pair32(q[i], p0, p1);
                best = fminf(best, e[i]);
            }
            float d[4];
            edge_pair32x2(A2[0], p0, p1, -p1.w, d[0], d[1]);
            edge_pair32x2(A2[1], p0, p1, -p1.w, d[2], d[3]);
            same = same && __float_as_uint(d[0]) == __float_as_uint(e[0]) &&
                   __float_as_uint(d[1]) == __float_as_uint(e[1]) && __float_as_uint(d[2]) == __float_as_uint(e[2]) &&
                   __float_as_uint(d[3]) == __float_as_uint(e[2]);
        }
        const double e = __longlong_as_double((long long)f32_as_f64_bits(best));
        d2[k] = same ? min_nn(v, e) : __longlong_as_double(0x7ff8000000000000ll);
    }
}

// gather planes of a Geom into per-face AoS records
__global__ void planes_to_aos(const double* __restrict__ planes, uint64_t n, uint64_t n_pad, double* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int f = 0; f < NF; ++f) out[NF * i + f] = planes[(uint64_t)f * n_pad + i];
}

// 8 independent DFMA chains per thread, 148 x 8 CTAs x 256 threads.
__global__ void __launch_bounds__(256) dfma_kernel(double* out, int iters, double s) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = fma(x[k], s, 0.5);
    }
    double acc = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += x[k];
    if (acc == 1234.5678) out[0] = acc;  // keep the chains alive
}

}  // namespace

void run_pairs(const Ctx& cx, const double* a9, const double* b9, uint64_t n, double* dist, uint8_t* hit) {
    const cudaStream_t st = cx.stream;
    if (n == 0) return;
    double *da = nullptr, *db = nullptr, *dd = nullptr;
    uint8_t* dh = nullptr;
    CK(cudaMallocAsync(&da, 9 * n * sizeof(double), st));
    CK(cudaMallocAsync(&db, 9 * n * sizeof(double), st));
    h2d(da, a9, 9 * n * sizeof(double), st);
    h2d(db, b9, 9 * n * sizeof(double), st);
    if (dist) CK(cudaMallocAsync(&dd, n * sizeof(double), st));
    if (hit) CK(cudaMallocAsync(&dh, n, st));
    pairs_kernel<<<(unsigned)std::min<uint64_t>((n + 127) / 128, 148 * 16), 128, 0, st>>>(da, db, n, dd, dh);
    CK(cudaGetLastError());
    if (dist) CK(cudaMemcpyAsync(dist, dd, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (hit) CK(cudaMemcpyAsync(hit, dh, n, cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(da, st));
    CK(cudaFreeAsync(db, st));
    if (dd) CK(cudaFreeAsync(dd, st));
    if (dh) CK(cudaFreeAsync(dh, st));
    CK(cudaStreamSynchronize(st));
}

void run_pairs_filter(const Ctx& cx, const Geom& A, const Geom& B, double* d2, const double* origin) {
    const cudaStream_t st = cx.stream;
    const uint64_t n = A.n;
    if (n == 0) return;
    double *pa = nullptr, *pb = nullptr, *dd = nullptr;
    CK(cudaMallocAsync(&pa, NF * n * sizeof(double), st));
    CK(cudaMallocAsync(&pb, NF * n * sizeof(double), st));
    CK(cudaMallocAsync(&dd, n * sizeof(double), st));
    planes_to_aos<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(A.planes, n, A.n_pad, pa);
    planes_to_aos<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(B.planes, n, B.n_pad, pb);
    const unsigned grid = (unsigned)std::min<uint64_t>((n + 127) / 128, 148 * 16);
    if (origin)
        filter_pairs_f32_kernel<<<grid, 128, 0, st>>>(pa, pb, n, origin[0], origin[1], origin[2], dd);
    else
        filter_pairs_kernel<<<grid, 128, 0, st>>>(pa, pb, n, dd);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(d2, dd, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(pa, st));
    CK(cudaFreeAsync(pb, st));
    CK(cudaFreeAsync(dd, st));
    CK(cudaStreamSynchronize(st));
}

double fp64_peak(const Ctx& cx, double* ms_out) {
    const cudaStream_t st = cx.stream;
    double* out = nullptr;
    CK(cudaMallocAsync(&out, sizeof(double), st));
    const int blocks = cx.sms * 8, threads = 256, iters = 4096;
    EventPair& evs = thread_events();
    cudaEvent_t e0 = evs.e[0], e1 = evs.e[1];
    dfma_kernel<<<blocks, threads, 0, st>>>(out, 64, 0.999);  // warm-up
    CK(cudaEventRecord(e0, st));
    dfma_kernel<<<blocks, threads, 0, st>>>(out, iters, 0.999);
    CK(cudaEventRecord(e1, st));
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    CK(cudaFreeAsync(out, st));
    CK(cudaStreamSynchronize(st));
    if (ms_out) *ms_out = ms;
    const double flops = 2.0 * 16 * 8 * (double)iters * blocks * threads;
    return flops / (ms * 1e-3) / 1e12;
}

}  // namespace tdb
