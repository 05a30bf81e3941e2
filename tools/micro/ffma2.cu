// microbenchmark: FP32 FMA throughput, scalar FFMA vs packed FFMA2 (sm_100a)
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, float a, float b, int iters) {
    float x[16];
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3f + i;
    if (MODE == 0) {
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], a, b);
    } else {
        float2* y = reinterpret_cast<float2*>(x);
        const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int i = 0; i < 8; ++i) y[i] = __ffma2_rn(y[i], a2, b2);
    }
    float s = 0.f;
    for (int i = 0; i < 16; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float* d;
    const int blocks = 148 * 8, threads = 256, iters = 20000;
    cudaMalloc(&d, blocks * threads * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<blocks, threads>>>(d, 0.999f, 1e-4f, iters);
            else k<1><<<blocks, threads>>>(d, 0.999f, 1e-4f, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double flops = 2.0 * 16 * (double)iters * blocks * threads;
            if (rep == 2) printf("%s: %.2f TFLOP/s (%.3f ms)\n", mode ? "FFMA2" : "FFMA ", flops / ms / 1e9, ms);
        }
    }
    return 0;
}
