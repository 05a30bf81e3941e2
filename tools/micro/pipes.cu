// microbenchmark: issue cost of FP32 FMA forms on sm_100a and whether ALU work overlaps them.
//   A: scalar FFMA, all-register operands      B: packed FFMA2, all-register operands
//   C: FFMA2 + an independent LOP3/IADD3 chain  D: scalar FFMA + the same ALU chain
//   E: ALU chain alone
// Reported per kernel: time and warp-instructions of each kind per SMSP-cycle.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, unsigned* iout, int iters, float s) {
    float x[16], y[16];
    unsigned u[8];
    for (int i = 0; i < 16; ++i) {
        x[i] = threadIdx.x * 1e-3f + i;
        y[i] = s * (i + 1) + threadIdx.x * 1e-6f;  // registers, not constants
    }
    for (int i = 0; i < 8; ++i) u[i] = threadIdx.x * 7u + i;
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0 || MODE == 3) {
#pragma unroll
            for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], y[i], y[15 - i]);
        }
        if (MODE == 1 || MODE == 2) {
            float2* xx = reinterpret_cast<float2*>(x);
            float2* yy = reinterpret_cast<float2*>(y);
#pragma unroll
            for (int i = 0; i < 8; ++i) xx[i] = __ffma2_rn(xx[i], yy[i], yy[7 - i]);
        }
        if (MODE >= 2) {
#pragma unroll
            for (int i = 0; i < 8; ++i) u[i] = ((u[i] ^ (u[(i + 1) & 7] >> 3)) + 0x9e3779b9u) | (u[i] << 1);
        }
    }
    float t = 0.f;
    for (int i = 0; i < 16; ++i) t += x[i];
    unsigned v = 0;
    for (int i = 0; i < 8; ++i) v ^= u[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
    iout[blockIdx.x * blockDim.x + threadIdx.x] = v;
}

int main() {
    float* d;
    unsigned* di;
    const int blocks = 148 * 8, threads = 256, iters = 20000;
    cudaMalloc(&d, blocks * threads * 4);
    cudaMalloc(&di, blocks * threads * 4);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[5] = {"A scalar FFMA (reg)", "B FFMA2 (reg)", "C FFMA2 + ALU", "D FFMA + ALU", "E ALU only"};
    for (int mode = 0; mode < 5; ++mode) {
        float ms = 0.f;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            switch (mode) {
            case 0: k<0><<<blocks, threads>>>(d, di, iters, 1e-4f); break;
            case 1: k<1><<<blocks, threads>>>(d, di, iters, 1e-4f); break;
            case 2: k<2><<<blocks, threads>>>(d, di, iters, 1e-4f); break;
            case 3: k<3><<<blocks, threads>>>(d, di, iters, 1e-4f); break;
            default: k<4><<<blocks, threads>>>(d, di, iters, 1e-4f); break;
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
        }
        const double fl = (mode == 4) ? 0.0 : 2.0 * 16 * (double)iters * blocks * threads;
        printf("%-22s %8.3f ms  %6.2f TFLOP/s\n", names[mode], ms, fl / ms / 1e9);
    }
    return 0;
}
