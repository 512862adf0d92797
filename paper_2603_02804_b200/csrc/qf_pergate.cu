// Per-gate (unfused) comparator: one HBM traversal per gate — the
// reference's naive path (engine.cpp:757-894) with psi uncomputed in place
// instead of a stored ledger. BASELINE config 5's "unfused" kernels.
#include "qf_device.cuh"

namespace qfb {
namespace {

// ------------------------------------------ per-gate (unfused) comparator
// One HBM traversal per gate: apply_rotation_kernel / apply_cz_kernel /
// apply_cnot_kernel (engine.cpp:111-202) and rotation_backward_kernel
// (engine.cpp:207-256), psi uncomputed in place instead of a stored ledger.
__device__ __forceinline__ void pair_apply_f(int axis, float c, float s, float2 &a, float2 &b) {
    const float2 A = a, Bv = b;
    switch (axis) {
    case 0:
        a = make_float2(c * A.x + s * Bv.y, c * A.y - s * Bv.x);
        b = make_float2(c * Bv.x + s * A.y, c * Bv.y - s * A.x);
        break;
    case 1:
        a = make_float2(c * A.x - s * Bv.x, c * A.y - s * Bv.y);
        b = make_float2(s * A.x + c * Bv.x, s * A.y + c * Bv.y);
        break;
    default:
        a = make_float2(c * A.x + s * A.y, c * A.y - s * A.x);
        b = make_float2(c * Bv.x - s * Bv.y, c * Bv.y + s * Bv.x);
        break;
    }
}

__global__ void __launch_bounds__(256) gate_fwd_kernel(float2 *psi, int n, uint64_t total_pairs,
                                                       int kind, int axis, uint32_t q0, uint32_t q1,
                                                       const double *theta, uint32_t param) {
    float c = 1.f, s = 0.f;
    if (kind == 0) {
        double sd, cd;
        sincos(theta[param] / 2.0, &sd, &cd);
        c = float(cd);
        s = float(sd);
    }
    const uint64_t half = 1ull << (n - 1);
    const uint32_t tq = kind == 0 ? q0 : q1;
    const uint64_t mask = 1ull << tq, lo = mask - 1;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total_pairs;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t smp = i / half, k = i % half;
        float2 *base = psi + (smp << n);
        const uint64_t i0 = ((k & ~lo) << 1) | (k & lo), i1 = i0 | mask;
        float2 a = base[i0], b = base[i1];
        if (kind == 0) {
            pair_apply_f(axis, c, s, a, b);
        } else if (kind == 1) { // CZ(q0,q1): -1 on |..1..1..> (target bit q1 = 1 in i1)
            if ((i1 >> q0) & 1ull) b = make_float2(-b.x, -b.y);
        } else { // CNOT: swap the pair when the control is set
            if ((i0 >> q0) & 1ull) {
                const float2 t = a;
                a = b;
                b = t;
            }
        }
        base[i0] = a;
        base[i1] = b;
    }
}

__global__ void __launch_bounds__(256) gate_bwd_kernel(float2 *psi, float2 *lam, int n,
                                                       uint64_t total_pairs, int kind, int axis,
                                                       uint32_t q0, uint32_t q1,
                                                       const double *theta, uint32_t param,
                                                       double *gpart) {
    float c = 1.f, s = 0.f;
    double sd = 0, cd = 1;
    if (kind == 0) {
        sincos(theta[param] / 2.0, &sd, &cd);
        c = float(cd);
        s = float(sd);
    }
    const float dc = float(-0.5 * sd), ds = float(0.5 * cd);
    const uint64_t half = 1ull << (n - 1);
    const uint32_t tq = kind == 0 ? q0 : q1;
    const uint64_t mask = 1ull << tq, lo = mask - 1;
    double acc = 0.0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total_pairs;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t smp = i / half, k = i % half;
        float2 *pb = psi + (smp << n), *lb = lam + (smp << n);
        const uint64_t i0 = ((k & ~lo) << 1) | (k & lo), i1 = i0 | mask;
        float2 a = pb[i0], b = pb[i1], la = lb[i0], lbv = lb[i1];
        if (kind == 0) {
            pair_apply_f(axis, c, -s, a, b); // psi_in = u^dag psi_out
            float2 wa = a, wb = b;
            pair_apply_f(axis, dc, ds, wa, wb); // du psi_in
            acc += double(la.x) * wa.x + double(la.y) * wa.y + double(lbv.x) * wb.x +
                   double(lbv.y) * wb.y;
            pair_apply_f(axis, c, -s, la, lbv);
        } else if (kind == 1) {
            if ((i1 >> q0) & 1ull) {
                b = make_float2(-b.x, -b.y);
                lbv = make_float2(-lbv.x, -lbv.y);
            }
        } else {
            if ((i0 >> q0) & 1ull) {
                float2 t = a; a = b; b = t;
                t = la; la = lbv; lbv = t;
            }
        }
        pb[i0] = a;
        pb[i1] = b;
        lb[i0] = la;
        lb[i1] = lbv;
    }
    if (kind == 0) {
        __shared__ double red[8];
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < 8; ++w) t += red[w];
            gpart[blockIdx.x] = t;
        }
    }
}

__global__ void gate_grad_reduce_kernel(const double *gpart, int gblocks, const uint32_t *params,
                                        int n_rot, double *grad) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rot) return;
    double s = 0.0;
    for (int b = 0; b < gblocks; ++b) s += gpart[size_t(r) * gblocks + b];
    grad[params[r]] = s;
}

} // namespace

int gate_grid(uint64_t pairs) {
    uint64_t b = (pairs + 255) / 256;
    if (b > 148 * 8) b = 148 * 8;
    return int(b ? b : 1);
}

cudaError_t launch_gate_fwd(cudaStream_t st, float2 *psi, int n, uint32_t batch, int kind,
                            int axis, uint32_t q0, uint32_t q1, const double *theta,
                            uint32_t param) {
    const uint64_t pairs = (uint64_t(batch) << n) / 2;
    gate_fwd_kernel<<<gate_grid(pairs), 256, 0, st>>>(psi, n, pairs, kind, axis, q0, q1, theta, param);
    return cudaGetLastError();
}

cudaError_t launch_gate_bwd(cudaStream_t st, float2 *psi, float2 *lam, int n, uint32_t batch,
                            int kind, int axis, uint32_t q0, uint32_t q1, const double *theta,
                            uint32_t param, double *gpart) {
    const uint64_t pairs = (uint64_t(batch) << n) / 2;
    gate_bwd_kernel<<<gate_grid(pairs), 256, 0, st>>>(psi, lam, n, pairs, kind, axis, q0, q1, theta,
                                                      param, gpart);
    return cudaGetLastError();
}

cudaError_t launch_gate_grad_reduce(cudaStream_t st, const double *gpart, int gblocks,
                                    const uint32_t *params, int n_rot, double *grad) {
    if (n_rot == 0) return cudaSuccess;
    gate_grad_reduce_kernel<<<(n_rot + 127) / 128, 128, 0, st>>>(gpart, gblocks, params, n_rot, grad);
    return cudaGetLastError();
}

} // namespace qfb
