// Micro-probe: FFMA vs FFMA2 (packed f32x2) throughput on this B200.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float *out, int iters, float a, float b) {
    float x[16];
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
            if (MODE == 0) {
                x[i] = fmaf(x[i], a, b);
                x[i + 1] = fmaf(x[i + 1], a, b);
            } else {
                unsigned long long v = (unsigned long long)__float_as_uint(x[i]) |
                                       ((unsigned long long)__float_as_uint(x[i + 1]) << 32);
                unsigned long long av = (unsigned long long)__float_as_uint(a) |
                                        ((unsigned long long)__float_as_uint(a) << 32);
                unsigned long long bv = (unsigned long long)__float_as_uint(b) |
                                        ((unsigned long long)__float_as_uint(b) << 32);
                unsigned long long r;
                asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(v), "l"(av), "l"(bv));
                x[i] = __uint_as_float(unsigned(r));
                x[i + 1] = __uint_as_float(unsigned(r >> 32));
            }
        }
    }
    float s = 0;
    for (int i = 0; i < 16; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float *o;
    cudaMalloc(&o, 148 * 8 * 256 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<148 * 8, 256>>>(o, iters, 0.999f, 1e-3f);
            else k<1><<<148 * 8, 256>>>(o, iters, 0.999f, 1e-3f);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double fma = 148.0 * 8 * 256 * iters * 16;
            printf("mode %s rep %d: %.3f ms  %.2f TFMA/s\n", mode ? "FFMA2" : "FFMA", rep, ms,
                   fma / ms / 1e9);
        }
    }
    return 0;
}
