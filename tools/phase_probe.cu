// Micro-probe (tooling, not product): throughput of the backward group-phase
// code of qf_device.cuh in isolation — no TMA, no HBM — to separate the cost
// of the phase arithmetic + barriers from the pipeline around it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2603_02804_b200/csrc \
//        -o phase_probe phase_probe.cu -lcuda
// Each CTA = 512 threads = two 256-thread halves, each on its own psi+lambda
// tile in shared memory, running the layout-A backward phase sequence
// (G2 R1, G1 R1, G0 R1+D+R0, G2 R0, G1 R0) `iters` times.
#include <cstdio>
#include <vector>

#include "qf_device.cuh"

using namespace qfb;
using namespace qfb::dev;

template <int G, uint32_t OPS, int M>
__device__ __forceinline__ void phase_var(uint8_t *pt, uint8_t *lt, uint32_t tau, const PhaseEnv &e,
                                          float2 (&p)[16], float2 (&l)[16]) {
    if (M != 2) { lds16<G>(pt, tau, p); lds16<G>(lt, tau, l); }
    if (M != 3) {
        if (OPS & 4u) {
            ry_round<G, true, true>(p, e.rys + 12, e.rot, e.mgs[3 + G], e.scale);
            ry_round<G, true, true>(l, e.rys + 12, e.rot, e.mgs[3 + G], e.scale);
            kmeasure<G, true, false>(p, l, e.rot, e.acc_w + 12 * 8, 1.f);
        }
        if (OPS & 2u) { apply_diag<true>(p, e.d, e.treg_s); apply_diag<true>(l, e.d, e.treg_s); }
        if (OPS & 1u) {
            ry_round<G, true, true>(p, e.rys, e.rot, e.mgs[G], e.scale);
            ry_round<G, true, true>(l, e.rys, e.rot, e.mgs[G], e.scale);
            kmeasure<G, true, false>(p, l, e.rot, e.acc_w, 1.f);
        }
    }
    if (M != 2) { sts16<G>(pt, tau, p); sts16<G>(lt, tau, l); }
}
template <int M>
__global__ void __launch_bounds__(512, 1) probe_var(const DiagTab *dt, int iters, float *out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    float4 *rys = reinterpret_cast<float4 *>(smem + 4 * kTileBytes);
    float2 *treg_s = reinterpret_cast<float2 *>(rys + 24);
    float2 *mgs = treg_s + 16;
    double *acc = reinterpret_cast<double *>(mgs + 8);
    const uint32_t tid = threadIdx.x, half = tid >> 8, gtid = tid & 255u, warp = tid >> 5;
    if (tid < 24) rys[tid] = ry_entry(make_float2(0.9f + 0.001f * tid, 0.3f));
    if (tid < 16) treg_s[tid] = dt->treg[tid];
    if (tid < 6) mgs[tid] = make_float2(0.7f, 0.7f);
    for (uint32_t i = tid; i < 16 * 2 * 12 * 8; i += 512) acc[i] = 0.0;
    uint8_t *pt = smem + half * 2 * kTileBytes;
    for (uint32_t i = gtid; i < 2 * kTileAmps; i += 256)
        reinterpret_cast<float2 *>(pt)[i] = make_float2(1e-3f * (i & 7), 1e-3f);
    __syncthreads();
    PhaseEnv env;
    env.rys = rys; env.mgs = mgs; env.rot = 0xFFFu; env.scale = false; env.kc = nullptr; env.zm = 0;
    env.treg_s = treg_s; env.acc_w = acc + warp * 2 * 12 * 8;
    env.d = diag_ctx(gtid, dt->tthr[gtid], 0u, dt, nullptr, nullptr, blockIdx.x & 255u);
    float2 p[16], l[16];
    for (int j = 0; j < 16; ++j) { p[j] = make_float2(1e-3f * j, gtid * 1e-6f); l[j] = p[j]; }
    uint8_t *lt = pt + kTileBytes;
    for (int it = 0; it < iters; ++it) {
        phase_var<2, 4, M>(pt, lt, gtid, env, p, l);
        asm volatile("bar.sync %0, 256;" ::"r"(1 + int(half)) : "memory");
        phase_var<1, 4, M>(pt, lt, gtid, env, p, l);
        asm volatile("bar.sync %0, 256;" ::"r"(1 + int(half)) : "memory");
        phase_var<0, 7, M>(pt, lt, gtid, env, p, l);
        asm volatile("bar.sync %0, 256;" ::"r"(1 + int(half)) : "memory");
        phase_var<2, 1, M>(pt, lt, gtid, env, p, l);
        asm volatile("bar.sync %0, 256;" ::"r"(1 + int(half)) : "memory");
        phase_var<1, 1, M>(pt, lt, gtid, env, p, l);
        asm volatile("bar.sync %0, 256;" ::"r"(1 + int(half)) : "memory");
    }
    __syncthreads();
    float s = 0;
    for (int j = 0; j < 16; ++j) s += p[j].x + l[j].y;
    if (tid == 0) out[blockIdx.x] = float(acc[0]) + reinterpret_cast<float *>(pt)[5] + s;
    else if (s == 123.f) out[1] = s;
}

template <int MODE, bool SCALE = true, int SKEW = 0> // MODE 0 = named barriers between phases, 1 = none (timing only)
__global__ void __launch_bounds__(512, 1) probe(const DiagTab *dt, int iters, float *out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    float4 *rys = reinterpret_cast<float4 *>(smem + 4 * kTileBytes);
    float2 *treg_s = reinterpret_cast<float2 *>(rys + 24);
    float2 *mgs = treg_s + 16;
    double *acc = reinterpret_cast<double *>(mgs + 8);
    const uint32_t tid = threadIdx.x, half = tid >> 8, gtid = tid & 255u, warp = tid >> 5;
    if (tid < 24) rys[tid] = ry_entry(make_float2(0.9f + 0.001f * tid, 0.3f));
    if (tid < 16) treg_s[tid] = dt->treg[tid];
    if (tid < 6) mgs[tid] = make_float2(0.7f, 0.7f);
    for (uint32_t i = tid; i < 16 * 2 * 12 * 8; i += 512) acc[i] = 0.0;
    uint8_t *pt = smem + half * 2 * kTileBytes;
    for (uint32_t i = gtid; i < 2 * kTileAmps; i += 256)
        reinterpret_cast<float2 *>(pt)[i] = make_float2(1e-3f * (i & 7), 1e-3f);
    __syncthreads();
    PhaseEnv env;
    env.rys = rys;
    env.mgs = mgs;
    env.rot = 0xFFFu;
    env.scale = SCALE;
    env.kc = nullptr;
    env.zm = 0;
    env.treg_s = treg_s;
    env.acc_w = acc + warp * 2 * 12 * 8;
    env.d = diag_ctx(gtid, dt->tthr[gtid], 0u, dt, nullptr, nullptr, blockIdx.x & 255u);
    if (SKEW && half) { // start half 1 SKEW cycles late
        const long long t0 = clock64();
        while (clock64() - t0 < SKEW) {}
    }
    const int G[5] = {1, 2, 0, 1, 2};
    const int O[5] = {1, 1, 7, 4, 4};
    for (int it = 0; it < iters; ++it) {
        for (int i = 4; i >= 0; --i) {
            if (MODE == 0 && i != 4) asm volatile("bar.sync %0, 256;" ::"r"(1 + int(half)) : "memory");
            run_phase_bwd(G[i], pt, pt + kTileBytes, gtid, O[i], env);
        }
        if (MODE == 0) asm volatile("bar.sync %0, 256;" ::"r"(1 + int(half)) : "memory");
    }
    __syncthreads();
    if (tid == 0) out[blockIdx.x] = float(acc[0]) + reinterpret_cast<float *>(pt)[5];
}

// pure FFMA2 at this kernel's occupancy (512 threads/SM), `CH` independent chains
template <int CH>
__global__ void __launch_bounds__(512, 1) ffma2_occ(float *out, int iters) {
    float2 x[CH];
    for (int i = 0; i < CH; ++i) x[i] = make_float2(threadIdx.x * 1e-3f + i, i);
    const float2 a = make_float2(0.999f, 0.999f), b = make_float2(1e-3f, 1e-3f);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int r = 0; r < 32 / CH; ++r)
#pragma unroll
            for (int i = 0; i < CH; ++i) x[i] = __ffma2_rn(x[i], a, b);
    float s = 0;
    for (int i = 0; i < CH; ++i) s += x[i].x + x[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH> void run_occ(float *o) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        ffma2_occ<CH><<<148, 512>>>(o, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("FFMA2 512 thr/SM, %2d chains: %.2f TFMA/s\n", CH, 148.0 * 512 * iters * 64 / ms / 1e9);
    }
}

int main() {
    DiagTab h{};
    for (int i = 0; i < 16; ++i) h.treg[i] = make_float2(0.6f, 0.8f);
    for (int i = 0; i < 256; ++i) h.tthr[i] = h.tt1[i] = h.tt2[i] = make_float2(0.8f, 0.6f);
    DiagTab *d;
    float *o;
    cudaMalloc(&d, sizeof(DiagTab));
    cudaMalloc(&o, 148 * 512 * 4);
    run_occ<2>(o);
    run_occ<4>(o);
    run_occ<8>(o);
    run_occ<16>(o);
    cudaMemcpy(d, &h, sizeof(h), cudaMemcpyHostToDevice);
    const size_t smem = 4 * kTileBytes + 24 * 16 + 16 * 8 + 8 * 8 + 16 * 2 * 12 * 8 * 8 + 1024;
    cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 200;
    cudaFuncSetAttribute(probe<0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(probe<0, false, 2000>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(probe<0, false, 5000>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(probe<0, false, 12000>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    for (int sk = 0; sk < 3; ++sk) {
        cudaEventRecord(e0);
        if (sk == 0) probe<0, false, 2000><<<148, 512, smem>>>(d, iters, o);
        if (sk == 1) probe<0, false, 5000><<<148, 512, smem>>>(d, iters, o);
        if (sk == 2) probe<0, false, 12000><<<148, 512, smem>>>(d, iters, o);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("skew %d: %.3f ms  %.1f us/tile/half\n", sk == 0 ? 2000 : sk == 1 ? 5000 : 12000, ms, ms * 1e3 / iters);
    }
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        probe<0, false><<<148, 512, smem>>>(d, iters, o);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("mode bar, scales folded: %.3f ms  %.1f us/tile/half\n", ms, ms * 1e3 / iters);
    }
    { // one half alone per SM (256 threads): how much do the two halves overlap?
        cudaFuncSetAttribute(probe_var<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            probe_var<1><<<148, 256, smem>>>(d, iters, o);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("one half per SM: %.1f us/tile\n", ms * 1e3 / iters);
        }
    }
    for (int m = 1; m <= 3; ++m) {
        if (m == 1) cudaFuncSetAttribute(probe_var<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (m == 2) cudaFuncSetAttribute(probe_var<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (m == 3) cudaFuncSetAttribute(probe_var<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (m == 1) probe_var<1><<<148, 512, smem>>>(d, iters, o);
            if (m == 2) probe_var<2><<<148, 512, smem>>>(d, iters, o);
            if (m == 3) probe_var<3><<<148, 512, smem>>>(d, iters, o);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("variant %s: %.1f us/tile/half\n", m == 1 ? "full" : m == 2 ? "compute only" : "smem only", ms * 1e3 / iters);
        }
    }
    for (int mode = 0; mode < 2; ++mode)
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            if (mode == 0) probe<0><<<148, 512, smem>>>(d, iters, o);
            else probe<1><<<148, 512, smem>>>(d, iters, o);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            // layout-A backward pass: 24 qubit-rounds x (2 Ry + 3 K) FFMA2 + 6 scale FMUL2
            // per amplitude = 252 lane-FMA (+ 16 diag)
            const double amps = 148.0 * 2 * iters * kTileAmps;
            printf("mode %s rep %d: %.3f ms  %.1f us/tile/half  %.2f TFMA/s (268 lane-FMA/amp)\n",
                   mode ? "nobar" : "bar", rep, ms, ms * 1e3 / iters, amps * 268 / ms / 1e9);
        }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
