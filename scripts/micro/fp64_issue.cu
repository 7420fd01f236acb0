// FP64 issue-model microbenchmarks (B200): cycles per warp instruction for
// DFMA/DMUL/DADD operand patterns, and whether ALU ops co-issue with FP64.
#include <cstdio>
#include <cuda_runtime.h>
#define N_IT 4096
template <int V>
__global__ void k(double* out, double s, int* iout) {
    double a0 = s + threadIdx.x, a1 = a0 * 1.1, a2 = a0 * 1.2, a3 = a0 * 1.3, a4 = a0 * 1.4, a5 = a0 * 1.5, a6 = a0 * 1.6, a7 = a0 * 1.7;
    double x0 = s * 0.5, x1 = s * 0.6, x2 = s * 0.7, x3 = s * 0.8, x4 = s * 0.9, x5 = s * 0.31, x6 = s * 0.32, x7 = s * 0.33;
    double y0 = s * 0.25, y1 = s * 0.26, y2 = s * 0.27, y3 = s * 0.28, y4 = s * 0.29, y5 = s * 0.21, y6 = s * 0.22, y7 = s * 0.23;
    int i0 = threadIdx.x, i1 = i0 + 1, i2 = i0 + 2, i3 = i0 + 3;
    float f0 = (float)s, f1 = f0 * 1.1f, f2 = f0 * 1.2f, f3 = f0 * 1.3f, g0 = f0 * 0.5f, g1 = f0 * 0.6f, g2 = f0 * 0.7f,
          g3 = f0 * 0.8f, h0 = f0 * 0.25f, h1 = f0 * 0.26f, h2 = f0 * 0.27f, h3 = f0 * 0.28f;
#pragma unroll 1
    for (int it = 0; it < N_IT; ++it) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (V == 0) {  // DFMA, 3 distinct registers (acc, x, y)
                a0 = fma(x0, y0, a0); a1 = fma(x1, y1, a1); a2 = fma(x2, y2, a2); a3 = fma(x3, y3, a3);
                a4 = fma(x4, y4, a4); a5 = fma(x5, y5, a5); a6 = fma(x6, y6, a6); a7 = fma(x7, y7, a7);
            } else if (V == 1) {  // DFMA, shared multiplier x0 (reuse)
                a0 = fma(x0, y0, a0); a1 = fma(x0, y1, a1); a2 = fma(x0, y2, a2); a3 = fma(x0, y3, a3);
                a4 = fma(x0, y4, a4); a5 = fma(x0, y5, a5); a6 = fma(x0, y6, a6); a7 = fma(x0, y7, a7);
            } else if (V == 2) {  // DMUL-like 2 operand: a = a * x
                a0 = a0 * x0; a1 = a1 * x1; a2 = a2 * x2; a3 = a3 * x3; a4 = a4 * x4; a5 = a5 * x5; a6 = a6 * x6; a7 = a7 * x7;
            } else if (V == 3) {  // DFMA 3 distinct + 1 int op per DFMA
                a0 = fma(x0, y0, a0); i0 = max(i0, __double2hiint(a0)); a1 = fma(x1, y1, a1); i1 = max(i1, __double2hiint(a1));
                a2 = fma(x2, y2, a2); i2 = max(i2, __double2hiint(a2)); a3 = fma(x3, y3, a3); i3 = max(i3, __double2hiint(a3));
                a4 = fma(x4, y4, a4); i0 = max(i0, __double2hiint(a4)); a5 = fma(x5, y5, a5); i1 = max(i1, __double2hiint(a5));
                a6 = fma(x6, y6, a6); i2 = max(i2, __double2hiint(a6)); a7 = fma(x7, y7, a7); i3 = max(i3, __double2hiint(a7));
            } else if (V == 4) {  // DMUL 2 operand + 1 int op
                a0 = a0 * x0; i0 = max(i0, __double2hiint(a0)); a1 = a1 * x1; i1 = max(i1, __double2hiint(a1));
                a2 = a2 * x2; i2 = max(i2, __double2hiint(a2)); a3 = a3 * x3; i3 = max(i3, __double2hiint(a3));
                a4 = a4 * x4; i0 = max(i0, __double2hiint(a4)); a5 = a5 * x5; i1 = max(i1, __double2hiint(a5));
                a6 = a6 * x6; i2 = max(i2, __double2hiint(a6)); a7 = a7 * x7; i3 = max(i3, __double2hiint(a7));
            } else if (V == 5) {  // DFMA with the accumulator as multiplicand: a = fma(a, x, y) (3 distinct)
                a0 = fma(a0, x0, y0); a1 = fma(a1, x1, y1); a2 = fma(a2, x2, y2); a3 = fma(a3, x3, y3);
                a4 = fma(a4, x4, y4); a5 = fma(a5, x5, y5); a6 = fma(a6, x6, y6); a7 = fma(a7, x7, y7);
            } else if (V == 6) {  // DFMA a = fma(a, x, a)  (2 distinct)
                a0 = fma(a0, x0, a0); a1 = fma(a1, x1, a1); a2 = fma(a2, x2, a2); a3 = fma(a3, x3, a3);
                a4 = fma(a4, x4, a4); a5 = fma(a5, x5, a5); a6 = fma(a6, x6, a6); a7 = fma(a7, x7, a7);
            } else if (V == 7) {  // DFMA 3 distinct + 2 int ops per DFMA
                a0 = fma(x0, y0, a0); i0 = max(i0, __double2hiint(a0)) ^ i1; a1 = fma(x1, y1, a1); i1 = max(i1, __double2hiint(a1)) ^ i2;
                a2 = fma(x2, y2, a2); i2 = max(i2, __double2hiint(a2)) ^ i3; a3 = fma(x3, y3, a3); i3 = max(i3, __double2hiint(a3)) ^ i0;
                a4 = fma(x4, y4, a4); i0 = max(i0, __double2hiint(a4)) ^ i1; a5 = fma(x5, y5, a5); i1 = max(i1, __double2hiint(a5)) ^ i2;
                a6 = fma(x6, y6, a6); i2 = max(i2, __double2hiint(a6)) ^ i3; a7 = fma(x7, y7, a7); i3 = max(i3, __double2hiint(a7)) ^ i0;
            } else if (V == 8) {  // DFMA 3 distinct + 1 FFMA 3 distinct
                a0 = fma(x0, y0, a0); f0 = fmaf(g0, h0, f0); a1 = fma(x1, y1, a1); f1 = fmaf(g1, h1, f1);
                a2 = fma(x2, y2, a2); f2 = fmaf(g2, h2, f2); a3 = fma(x3, y3, a3); f3 = fmaf(g3, h3, f3);
                a4 = fma(x4, y4, a4); f0 = fmaf(g1, h2, f0); a5 = fma(x5, y5, a5); f1 = fmaf(g2, h3, f1);
                a6 = fma(x6, y6, a6); f2 = fmaf(g3, h0, f2); a7 = fma(x7, y7, a7); f3 = fmaf(g0, h1, f3);
            } else if (V == 9) {  // FFMA only (8 per "fp64" slot count)
                f0 = fmaf(g0, h0, f0); f1 = fmaf(g1, h1, f1); f2 = fmaf(g2, h2, f2); f3 = fmaf(g3, h3, f3);
                f0 = fmaf(g1, h2, f0); f1 = fmaf(g2, h3, f1); f2 = fmaf(g3, h0, f2); f3 = fmaf(g0, h1, f3);
            } else if (V == 10) {  // DMUL + 1 FFMA
                a0 = a0 * x0; f0 = fmaf(g0, h0, f0); a1 = a1 * x1; f1 = fmaf(g1, h1, f1);
                a2 = a2 * x2; f2 = fmaf(g2, h2, f2); a3 = a3 * x3; f3 = fmaf(g3, h3, f3);
                a4 = a4 * x4; f0 = fmaf(g1, h2, f0); a5 = a5 * x5; f1 = fmaf(g2, h3, f1);
                a6 = a6 * x6; f2 = fmaf(g3, h0, f2); a7 = a7 * x7; f3 = fmaf(g0, h1, f3);
            } else if (V == 11) {  // DFMA 3 distinct + 1 IADD3 on even regs (not hi words)
                a0 = fma(x0, y0, a0); i0 = i0 + i1 + i2; a1 = fma(x1, y1, a1); i1 = i1 + i2 + i3;
                a2 = fma(x2, y2, a2); i2 = i2 + i3 + i0; a3 = fma(x3, y3, a3); i3 = i3 + i0 + i1;
                a4 = fma(x4, y4, a4); i0 = i0 + i1 + i2; a5 = fma(x5, y5, a5); i1 = i1 + i2 + i3;
                a6 = fma(x6, y6, a6); i2 = i2 + i3 + i0; a7 = fma(x7, y7, a7); i3 = i3 + i0 + i1;
            }
        }
        x0 = __hiloint2double(__double2hiint(x0) ^ (it & 1), __double2loint(x0));
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    iout[blockIdx.x * blockDim.x + threadIdx.x] = i0 + i1 + i2 + i3 + (int)(f0 + f1 + f2 + f3);
}
template <int V>
void run(const char* name, int nint_per_fp) {
    double* out; int* io;
    const int blocks = 148 * 8, threads = 256;
    cudaMalloc(&out, blocks * threads * 8); cudaMalloc(&io, blocks * threads * 4);
    k<V><<<blocks, threads>>>(out, 1.0, io);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k<V><<<blocks, threads>>>(out, 1.0, io);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double warp_fp = 5.0 * blocks * threads / 32 * N_IT * 32;  // fp64 warp-instr
    const double cyc = ms * 1e-3 * clk * 1e3 * 148 * 4;  // SMSP-cycles
    printf("%-40s %6.3f SMSP-cycles per FP64 warp instr  (%.2f TFLOP-eq)\n", name, cyc / warp_fp,
           warp_fp * 32 * 2 / (ms * 1e-3) / 1e12);
    cudaFree(out); cudaFree(io);
}
int main() {
    run<0>("DFMA 3 distinct", 0);
    run<1>("DFMA shared multiplier", 0);
    run<2>("DMUL 2 distinct", 0);
    run<3>("DFMA 3 distinct + 1 ALU", 1);
    run<4>("DMUL + 1 ALU", 1);
    run<5>("DFMA a=fma(a,x,y)", 0);
    run<6>("DFMA a=fma(a,x,a)", 0);
    run<7>("DFMA 3 distinct + 2 ALU", 2);
    run<8>("DFMA 3 distinct + 1 FFMA", 1);
    run<9>("FFMA only (per FFMA)", 0);
    run<10>("DMUL + 1 FFMA", 1);
    run<11>("DFMA 3 distinct + 1 IADD3", 1);
    return 0;
}
