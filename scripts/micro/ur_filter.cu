// Experiment: B faces as kernel parameters (constant bank, compile-time
// offsets after full unroll) so ptxas can feed them to DFMAs from uniform
// registers / the constant bank instead of vector registers. Measures
// pairs/s of the production pair_d2 (fast_pair.cuh) in that arrangement.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include
//        -I../../paper_1808_09571_b200/csrc -DNBF=16 ur_filter.cu -o ur_filter
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "fast_pair.cuh"

using namespace tdb;

#ifndef NBF
#define NBF 16
#endif

struct BGroup {
    double f[NBF][kFilterPlanes];
};

struct ParamFace {
    const BGroup* g;
    int q;
    const double* p;  // the same face in HBM (pierce_slow)
    uint64_t stride;
    __device__ __forceinline__ double operator()(int f) const { return g->f[q][f]; }
};

__global__ void __launch_bounds__(128, MINB) ur_kernel(const double* __restrict__ Ap, uint64_t An_pad, uint64_t n_rows,
                                                       const double* Bp, uint64_t Bn_pad, uint64_t bj0,
                                                       const __grid_constant__ BGroup g, double* out) {
    for (uint64_t row = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n_rows;
         row += (uint64_t)gridDim.x * blockDim.x) {
        AFace A;
        load_aface(A, FaceRefLdg{Ap + row, An_pad});
        double best = pos_inf();
#pragma unroll
        for (int q = 0; q < NBF; ++q) {
            if (g.f[q][F_DEG] != 0.0) continue;
            best = min_nn(best, pair_d2(A, ParamFace{&g, q, Bp + bj0 + q, Bn_pad}, Ap + row, An_pad));
        }
        if (best < out[row]) out[row] = best;
    }
}

int main(int argc, char** argv) {
    const uint64_t n = argc > 1 ? atoll(argv[1]) : (1 << 20);
    const int launches = argc > 2 ? atoi(argv[2]) : 256;
    const uint64_t pad = n;
    // random well-formed planes: triangles in a box, derived fields as prep_kernel computes them
    std::vector<double> P((size_t)NF * pad, 0.0);
    srand(7);
    auto rnd = [] { return rand() / (double)RAND_MAX; };
    for (uint64_t i = 0; i < n; ++i) {
        double v[9];
        const double cx = rnd() * 1000, cy = rnd() * 1000, cz = rnd() * 400;
        for (int k = 0; k < 3; ++k) v[3 * k] = cx + rnd(), v[3 * k + 1] = cy + rnd(), v[3 * k + 2] = cz + rnd();
        double e[9], L[3];
        for (int j = 0; j < 3; ++j) {
            const int q = (j + 1) % 3;
            for (int c = 0; c < 3; ++c) e[3 * j + c] = v[3 * q + c] - v[3 * j + c];
            L[j] = e[3 * j] * e[3 * j] + e[3 * j + 1] * e[3 * j + 1] + e[3 * j + 2] * e[3 * j + 2];
        }
        const double a0 = e[0], a1 = e[1], a2 = e[2], b0 = -e[6], b1 = -e[7], b2 = -e[8];
        const double Nx = a1 * b2 - a2 * b1, Ny = a2 * b0 - a0 * b2, Nz = a0 * b1 - a1 * b0;
        const double N2 = Nx * Nx + Ny * Ny + Nz * Nz, inv = 1 / sqrt(N2), inv2 = 1 / N2;
        double f[NF] = {};
        for (int k = 0; k < 9; ++k) f[F_V + k] = v[k], f[F_E + k] = e[k];
        for (int k = 0; k < 3; ++k) f[F_L + k] = L[k], f[F_IL + k] = 1 / L[k];
        f[F_N] = Nx * inv, f[F_N + 1] = Ny * inv, f[F_N + 2] = Nz * inv;
        f[F_U] = (b1 * Nz - b2 * Ny) * inv2, f[F_U + 1] = (b2 * Nx - b0 * Nz) * inv2, f[F_U + 2] = (b0 * Ny - b1 * Nx) * inv2;
        f[F_W] = (Ny * a2 - Nz * a1) * inv2, f[F_W + 1] = (Nz * a0 - Nx * a2) * inv2, f[F_W + 2] = (Nx * a1 - Ny * a0) * inv2;
        for (int k = 0; k < NF; ++k) P[(size_t)k * pad + i] = f[k];
    }
    double *dP, *out;
    cudaMalloc(&dP, P.size() * 8);
    cudaMalloc(&out, n * 8);
    cudaMemcpy(dP, P.data(), P.size() * 8, cudaMemcpyHostToDevice);
    cudaMemset(out, 0x7f, n * 8);
    std::vector<BGroup> groups(launches);
    for (int l = 0; l < launches; ++l)
        for (int q = 0; q < NBF; ++q)
            for (int k = 0; k < kFilterPlanes; ++k) groups[l].f[q][k] = P[(size_t)k * pad + (l * NBF + q) % n];
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const unsigned grid = sms * MINB * 4;
    for (int l = 0; l < 4; ++l) ur_kernel<<<grid, 128>>>(dP, pad, n, dP, pad, 0, groups[l], out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int l = 0; l < launches; ++l) ur_kernel<<<grid, 128>>>(dP, pad, n, dP, pad, (uint64_t)l * NBF % n, groups[l], out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double pairs = (double)n * NBF * launches;
    printf("NBF %d MINB %d: %.4g pairs/s (%.3f ms per launch) err=%s\n", NBF, MINB, pairs / (ms * 1e-3), ms / launches,
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
