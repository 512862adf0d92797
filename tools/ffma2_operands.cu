// Micro-probe (tooling, not product): FFMA2 issue rate vs the number of fresh
// 64-bit source operands per instruction (register-file read bandwidth).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o ffma2_operands ffma2_operands.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 f2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

// V = 0: acc[i] = fma(x[i], CONST, acc[i])          (1 fresh + acc)
// V = 1: acc[i] = fma(x[i], y[i], acc[i])           (3 fresh pairs)
// V = 2: acc[i] = fma(x[i], y[i & ~3], acc[i])      (y reused across 4 consecutive)
// V = 3: x[i]   = fma(CONST, y[i], x[i])            (Ry-like: const + 2 fresh)
template <int V>
__global__ void __launch_bounds__(512, 1) k(float *out, int iters) {
    float2 x[16], y[16], acc[16];
    for (int i = 0; i < 16; ++i) {
        x[i] = make_float2(threadIdx.x * 1e-6f + i, i);
        y[i] = make_float2(1e-3f * i, 0.5f);
        acc[i] = make_float2(0.f, 0.f);
    }
    const float2 C = make_float2(0.999f, 1.001f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (V == 0) acc[i] = f2(x[i], C, acc[i]);
            if (V == 1) acc[i] = f2(x[i], y[i], acc[i]);
            if (V == 2) acc[i] = f2(x[i], y[i & ~3], acc[i]);
            if (V == 3) x[i] = f2(C, y[i], x[i]);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) { // keep inputs live and changing
            if (V != 3) x[i] = f2(x[i], C, y[i]);
        }
    }
    float s = 0;
    for (int i = 0; i < 16; ++i) s += x[i].x + acc[i].y + y[i].x;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int V> void run(float *o, const char *name) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k<V><<<148, 512>>>(o, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double ffma2 = 148.0 * 512 * iters * (V == 3 ? 16 : 32);
    printf("%-48s %.2f TFMA/s\n", name, ffma2 * 2 / best / 1e9);
}

int main() {
    float *o;
    cudaMalloc(&o, 148 * 512 * 4);
    run<0>(o, "acc = fma(x, CONST, acc) (+ x update)");
    run<1>(o, "acc = fma(x, y, acc), 3 fresh (+ x update)");
    run<2>(o, "acc = fma(x, y[i&~3], acc) (+ x update)");
    run<3>(o, "x = fma(CONST, y, x)");
    return 0;
}
