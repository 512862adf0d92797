// Micro-probe (tooling, not product): FFMA2 throughput of the operand patterns
// the backward phase code uses, at its occupancy (512 threads/SM). Every
// iteration applies the 4-bit Ry round to psi and lambda (so nothing can be
// hoisted) and then one K-measure variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2603_02804_b200/csrc \
//        -o ffma2_patterns ffma2_patterns.cu
#include <cstdio>

#include "qf_device.cuh"

using namespace qfb::dev;

// K = 0: none (Ry only)
// K = 1: kbit3 x 4 (swapped operands, 2 accumulator sets per output)
// K = 2: one accumulator set per output, FFMA2
// K = 3: scalar FFMA, two accumulators per output (no swaps needed)
// K = 4: FFMA2 on (psi, lambda) products with lambda pre-swapped once per round
template <int K>
__global__ void __launch_bounds__(512, 1) pat(float *out, int iters, float4 e) {
    float2 p[16], l[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        p[j] = make_float2(threadIdx.x * 1e-6f + j, 0.5f * j);
        l[j] = make_float2(0.25f * j, threadIdx.x * 1e-6f - j);
    }
    float acc[12];
#pragma unroll
    for (int i = 0; i < 12; ++i) acc[i] = 0.f;
    for (int it = 0; it < iters; ++it) {
        ry2<0, true>(p, e);
        ry2<1, true>(p, e);
        ry2<2, true>(p, e);
        ry2<3, true>(p, e);
        ry2<0, true>(l, e);
        ry2<1, true>(l, e);
        ry2<2, true>(l, e);
        ry2<3, true>(l, e);
        if (K == 1) {
            float2 ps[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) ps[j] = make_float2(p[j].y, p[j].x);
            float v[12];
            kbit3<0>(p, l, v + 0);
            kbit3<1>(p, l, v + 3);
            kbit3<2>(p, l, v + 6);
            kbit3<3>(p, l, v + 9);
#pragma unroll
            for (int i = 0; i < 12; ++i) acc[i] += v[i];
        }
        if (K == 2) {
            float2 bx[4], ay[4], bz[4];
#pragma unroll
            for (int b = 0; b < 4; ++b) bx[b] = ay[b] = bz[b] = make_float2(0.f, 0.f);
#pragma unroll
            for (int b = 0; b < 4; ++b)
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    if (j & (1 << b)) continue;
                    const int j1 = j | (1 << b);
                    const float2 ps0 = make_float2(p[j].y, p[j].x), ps1 = make_float2(p[j1].y, p[j1].x);
                    bz[b] = __ffma2_rn(ps0, l[j], bz[b]);
                    bz[b] = __ffma2_rn(make_float2(-ps1.x, -ps1.y), l[j1], bz[b]);
                    bx[b] = __ffma2_rn(ps0, l[j1], bx[b]);
                    bx[b] = __ffma2_rn(ps1, l[j], bx[b]);
                    ay[b] = __ffma2_rn(p[j], l[j1], ay[b]);
                    ay[b] = __ffma2_rn(make_float2(-p[j1].x, -p[j1].y), l[j], ay[b]);
                }
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                acc[3 * b] += bx[b].x - bx[b].y;
                acc[3 * b + 1] += ay[b].x + ay[b].y;
                acc[3 * b + 2] += bz[b].x - bz[b].y;
            }
        }
        if (K == 3) {
            float a[24];
#pragma unroll
            for (int i = 0; i < 24; ++i) a[i] = 0.f;
#pragma unroll
            for (int b = 0; b < 4; ++b)
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    if (j & (1 << b)) continue;
                    const int j1 = j | (1 << b);
                    float *A = a + 6 * b;
                    A[0] = fmaf(p[j].y, l[j].x, A[0]);
                    A[1] = fmaf(p[j].x, l[j].y, A[1]);
                    A[0] = fmaf(-p[j1].y, l[j1].x, A[0]);
                    A[1] = fmaf(-p[j1].x, l[j1].y, A[1]);
                    A[2] = fmaf(p[j].y, l[j1].x, A[2]);
                    A[3] = fmaf(p[j].x, l[j1].y, A[3]);
                    A[2] = fmaf(p[j1].y, l[j].x, A[2]);
                    A[3] = fmaf(p[j1].x, l[j].y, A[3]);
                    A[4] = fmaf(p[j].x, l[j1].x, A[4]);
                    A[5] = fmaf(p[j].y, l[j1].y, A[5]);
                    A[4] = fmaf(-p[j1].x, l[j].x, A[4]);
                    A[5] = fmaf(-p[j1].y, l[j].y, A[5]);
                }
#pragma unroll
            for (int i = 0; i < 12; ++i) acc[i] += (i % 3 == 2 ? a[2 * i] + a[2 * i + 1] : a[2 * i] - a[2 * i + 1]);
        }
        if (K == 4) { // products in pair-major order, all 4 bits interleaved
            float2 r[12];
#pragma unroll
            for (int i = 0; i < 12; ++i) r[i] = make_float2(0.f, 0.f);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    if (j & (1 << b)) continue;
                    const int j1 = j | (1 << b);
                    const float2 ps0 = make_float2(p[j].y, p[j].x), ps1 = make_float2(p[j1].y, p[j1].x);
                    r[3 * b + 2] = __ffma2_rn(ps0, l[j], r[3 * b + 2]);
                    r[3 * b + 0] = __ffma2_rn(ps0, l[j1], r[3 * b + 0]);
                    r[3 * b + 1] = __ffma2_rn(p[j], l[j1], r[3 * b + 1]);
                    r[3 * b + 2] = __ffma2_rn(make_float2(-ps1.x, -ps1.y), l[j1], r[3 * b + 2]);
                    r[3 * b + 0] = __ffma2_rn(ps1, l[j], r[3 * b + 0]);
                    r[3 * b + 1] = __ffma2_rn(make_float2(-p[j1].x, -p[j1].y), l[j], r[3 * b + 1]);
                }
            }
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                acc[3 * b] += r[3 * b].x - r[3 * b].y;
                acc[3 * b + 1] += r[3 * b + 1].x + r[3 * b + 1].y;
                acc[3 * b + 2] += r[3 * b + 2].x - r[3 * b + 2].y;
            }
        }
        if (K == 5) { // FFMA2, operand-reuse ordering, single acc set
            float2 r[12];
#pragma unroll
            for (int i = 0; i < 12; ++i) r[i] = make_float2(0.f, 0.f);
#pragma unroll
            for (int b = 0; b < 4; ++b)
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    if (j & (1 << b)) continue;
                    const int j1 = j | (1 << b);
                    const float2 ps0 = make_float2(p[j].y, p[j].x), ps1 = make_float2(p[j1].y, p[j1].x);
                    r[3 * b + 2] = __ffma2_rn(ps0, l[j], r[3 * b + 2]);
                    r[3 * b + 0] = __ffma2_rn(ps0, l[j1], r[3 * b + 0]);
                    r[3 * b + 1] = __ffma2_rn(p[j], l[j1], r[3 * b + 1]);
                    r[3 * b + 1] = __ffma2_rn(make_float2(-p[j1].x, -p[j1].y), l[j], r[3 * b + 1]);
                    r[3 * b + 0] = __ffma2_rn(ps1, l[j], r[3 * b + 0]);
                    r[3 * b + 2] = __ffma2_rn(make_float2(-ps1.x, -ps1.y), l[j1], r[3 * b + 2]);
                }
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                acc[3 * b] += r[3 * b].x - r[3 * b].y;
                acc[3 * b + 1] += r[3 * b + 1].x + r[3 * b + 1].y;
                acc[3 * b + 2] += r[3 * b + 2].x - r[3 * b + 2].y;
            }
        }
        if (K == 6) { // scalar FFMA, one accumulator per output
            float a[12];
#pragma unroll
            for (int i = 0; i < 12; ++i) a[i] = 0.f;
#pragma unroll
            for (int b = 0; b < 4; ++b)
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    if (j & (1 << b)) continue;
                    const int j1 = j | (1 << b);
                    float *A = a + 3 * b;
                    A[2] = fmaf(p[j].y, l[j].x, A[2]);
                    A[2] = fmaf(-p[j].x, l[j].y, A[2]);
                    A[2] = fmaf(-p[j1].y, l[j1].x, A[2]);
                    A[2] = fmaf(p[j1].x, l[j1].y, A[2]);
                    A[0] = fmaf(p[j].y, l[j1].x, A[0]);
                    A[0] = fmaf(-p[j].x, l[j1].y, A[0]);
                    A[0] = fmaf(p[j1].y, l[j].x, A[0]);
                    A[0] = fmaf(-p[j1].x, l[j].y, A[0]);
                    A[1] = fmaf(p[j].x, l[j1].x, A[1]);
                    A[1] = fmaf(p[j].y, l[j1].y, A[1]);
                    A[1] = fmaf(-p[j1].x, l[j].x, A[1]);
                    A[1] = fmaf(-p[j1].y, l[j].y, A[1]);
                }
#pragma unroll
            for (int i = 0; i < 12; ++i) acc[i] += a[i];
        }
        if (K == 7) { // Y by FFMA2 (no swap), X and Z by scalar FFMA
            float a[16];
            float2 y[4];
#pragma unroll
            for (int i = 0; i < 16; ++i) a[i] = 0.f;
#pragma unroll
            for (int b = 0; b < 4; ++b) y[b] = make_float2(0.f, 0.f);
#pragma unroll
            for (int b = 0; b < 4; ++b)
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    if (j & (1 << b)) continue;
                    const int j1 = j | (1 << b);
                    float *A = a + 4 * b;
                    A[0] = fmaf(p[j].y, l[j].x, A[0]);
                    A[1] = fmaf(p[j].x, l[j].y, A[1]);
                    A[0] = fmaf(-p[j1].y, l[j1].x, A[0]);
                    A[1] = fmaf(-p[j1].x, l[j1].y, A[1]);
                    A[2] = fmaf(p[j].y, l[j1].x, A[2]);
                    A[3] = fmaf(p[j].x, l[j1].y, A[3]);
                    A[2] = fmaf(p[j1].y, l[j].x, A[2]);
                    A[3] = fmaf(p[j1].x, l[j].y, A[3]);
                    y[b] = __ffma2_rn(p[j], l[j1], y[b]);
                    y[b] = __ffma2_rn(make_float2(-p[j1].x, -p[j1].y), l[j], y[b]);
                }
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                acc[3 * b] += a[4 * b] - a[4 * b + 1];
                acc[3 * b + 1] += y[b].x + y[b].y;
                acc[3 * b + 2] += a[4 * b + 2] - a[4 * b + 3];
            }
        }
        if (K == 10) { // lambda-major: l[j] reused in slot B by 12 consecutive FFMA2
            float2 r[12];
#pragma unroll
            for (int i = 0; i < 12; ++i) r[i] = make_float2(0.f, 0.f);
#pragma unroll
            for (int j = 0; j < 16; ++j)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int k = j ^ (1 << b);
                    const float2 psj = make_float2(p[j].y, p[j].x), psk = make_float2(p[k].y, p[k].x);
                    float2 &bx = r[3 * b], &ay = r[3 * b + 1], &bz = r[3 * b + 2];
                    if (!(j & (1 << b))) {
                        bz = __ffma2_rn(psj, l[j], bz);
                        bx = __ffma2_rn(psk, l[j], bx);
                        ay = __ffma2_rn(make_float2(-p[k].x, -p[k].y), l[j], ay);
                    } else {
                        bz = __ffma2_rn(make_float2(-psj.x, -psj.y), l[j], bz);
                        bx = __ffma2_rn(psk, l[j], bx);
                        ay = __ffma2_rn(p[k], l[j], ay);
                    }
                }
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                acc[3 * b] += r[3 * b].x - r[3 * b].y;
                acc[3 * b + 1] += r[3 * b + 1].x + r[3 * b + 1].y;
                acc[3 * b + 2] += r[3 * b + 2].x - r[3 * b + 2].y;
            }
        }
        if (K == 8 || K == 9) { // 8: no swaps/negations (timing only); 9: swaps, no negations (split acc)
            float2 r[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) r[i] = make_float2(0.f, 0.f);
#pragma unroll
            for (int b = 0; b < 4; ++b)
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    if (j & (1 << b)) continue;
                    const int j1 = j | (1 << b);
                    const float2 ps0 = K == 8 ? p[j] : make_float2(p[j].y, p[j].x);
                    const float2 ps1 = K == 8 ? p[j1] : make_float2(p[j1].y, p[j1].x);
                    r[4 * b + 0] = __ffma2_rn(ps0, l[j], r[4 * b + 0]);
                    r[4 * b + 3] = __ffma2_rn(ps1, l[j1], r[4 * b + 3]);
                    r[4 * b + 1] = __ffma2_rn(ps0, l[j1], r[4 * b + 1]);
                    r[4 * b + 1] = __ffma2_rn(ps1, l[j], r[4 * b + 1]);
                    r[4 * b + 2] = __ffma2_rn(p[j], l[j1], r[4 * b + 2]);
                    r[4 * b + 2] = __ffma2_rn(l[j], p[j1], r[4 * b + 2]);
                }
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                acc[3 * b] += r[4 * b + 1].x - r[4 * b + 1].y;
                acc[3 * b + 1] += r[4 * b + 2].x + r[4 * b + 2].y;
                acc[3 * b + 2] += (r[4 * b].x - r[4 * b].y) - (r[4 * b + 3].x - r[4 * b + 3].y);
            }
        }
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) s += p[j].x + l[j].y;
#pragma unroll
    for (int i = 0; i < 12; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int K> void run(float *o, const char *name) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4000;
    const double lane = 2.0 * 4 * 16 * 2 + (K ? 4.0 * 48 * 2 : 0.0);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        pat<K><<<148, 512>>>(o, iters, make_float4(0.01f, 0.01f, 1.f, 0.f));
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double ry_ms = 148.0 * 512 * iters * 256 / 37.0e9;
    printf("%-44s %.2f TFMA/s total; K part %.2f TFMA/s (Ry at 37)\n", name,
           148.0 * 512 * iters * lane / best / 1e9,
           K ? 148.0 * 512 * iters * 384 / (best - ry_ms) / 1e9 : 0.0);
}

int main() {
    float *o;
    cudaMalloc(&o, 148 * 512 * 4);
    run<0>(o, "Ry only (psi, lambda)");
    run<1>(o, "Ry + K kbit3 (2 acc sets)");
    run<2>(o, "Ry + K single acc set");
    run<3>(o, "Ry + K scalar FFMA");
    run<4>(o, "Ry + K pair-major, bits interleaved");
    run<5>(o, "Ry + K FFMA2 reuse order, single acc");
    run<6>(o, "Ry + K scalar, one acc per output");
    run<7>(o, "Ry + K hybrid (Y FFMA2, X/Z FFMA)");
    run<8>(o, "Ry + K FFMA2 no swap/neg (timing only)");
    run<9>(o, "Ry + K FFMA2 swaps, no negation");
    run<10>(o, "Ry + K lambda-major (l reused)");
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
