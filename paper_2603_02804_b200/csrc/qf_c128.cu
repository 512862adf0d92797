// complex128 path (the reference's double instantiations, engine.cpp:896-944,
// checkpoint.cpp:190-213): one HBM traversal per gate in fp64 — the per-gate
// schedule of engine.cpp:757-894 with psi uncomputed in place (unitary in
// fp64: the round-trip drift stays at the 1e-15 level, no slots needed).
//   gate_fwd_c128:  apply_rotation/cz/cnot_kernel      engine.cpp:111-202
//   gate_bwd_c128:  rotation_backward_kernel            engine.cpp:207-256
//                   (psi_in = u^dag psi_out, Re<lam|du|psi_in>, lam <- u^dag lam)
//   seed_c128:      expectation_kernel + seed_adjoint   engine.cpp:346-435
// Reductions are per block in fp64 and summed in a fixed order (deterministic).
#include "qf_internal.h"

namespace qfb {
namespace {

// pair_apply (engine.cpp:36-59): u = c I - i s P on (a, b) = (|..0..>, |..1..>).
__device__ __forceinline__ void pair_apply_d(int axis, double c, double s, double2 &a, double2 &b) {
    const double2 A = a, Bv = b;
    switch (axis) {
    case 0: // Rx: [[c, -is], [-is, c]]
        a = make_double2(c * A.x + s * Bv.y, c * A.y - s * Bv.x);
        b = make_double2(c * Bv.x + s * A.y, c * Bv.y - s * A.x);
        break;
    case 1: // Ry: [[c, -s], [s, c]]
        a = make_double2(c * A.x - s * Bv.x, c * A.y - s * Bv.y);
        b = make_double2(s * A.x + c * Bv.x, s * A.y + c * Bv.y);
        break;
    default: // Rz: diag(c - is, c + is)
        a = make_double2(c * A.x + s * A.y, c * A.y - s * A.x);
        b = make_double2(c * Bv.x - s * Bv.y, c * Bv.y + s * Bv.x);
        break;
    }
}

struct PairIdx {
    uint64_t i0, i1;
};
__device__ __forceinline__ PairIdx pair_of(uint64_t i, int n, uint32_t tq, uint64_t &smp) {
    const uint64_t half = 1ull << (n - 1), mask = 1ull << tq, lo = mask - 1;
    smp = i / half;
    const uint64_t k = i % half, i0 = ((k & ~lo) << 1) | (k & lo);
    return {i0, i0 | mask};
}

__global__ void __launch_bounds__(256) gate_fwd_c128(double2 *psi, int n, uint64_t pairs, int kind,
                                                     int axis, uint32_t q0, uint32_t q1,
                                                     const double *theta, uint32_t param) {
    double c = 1.0, s = 0.0;
    if (kind == 0) sincos(theta[param] / 2.0, &s, &c);
    const uint32_t tq = kind == 0 ? q0 : q1;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < pairs;
         i += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t smp;
        const PairIdx p = pair_of(i, n, tq, smp);
        double2 *base = psi + (smp << n);
        double2 a = base[p.i0], b = base[p.i1];
        if (kind == 0) {
            pair_apply_d(axis, c, s, a, b);
        } else if (kind == 1) { // CZ: -1 on |..1..1..> (engine.cpp:111-136)
            if ((p.i1 >> q0) & 1ull) b = make_double2(-b.x, -b.y);
        } else { // CNOT(control q0, target q1) (engine.cpp:142-170)
            if ((p.i0 >> q0) & 1ull) {
                const double2 t = a;
                a = b;
                b = t;
            }
        }
        base[p.i0] = a;
        base[p.i1] = b;
    }
}

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double red[8];
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
    return t;
}

__global__ void __launch_bounds__(256) gate_bwd_c128(double2 *psi, double2 *lam, int n, uint64_t pairs,
                                                     int kind, int axis, uint32_t q0, uint32_t q1,
                                                     const double *theta, uint32_t param,
                                                     double *gpart) {
    double c = 1.0, s = 0.0;
    if (kind == 0) sincos(theta[param] / 2.0, &s, &c);
    const double dc = -0.5 * s, ds = 0.5 * c; // rotation_derivative (circuit.cpp:76-87)
    const uint32_t tq = kind == 0 ? q0 : q1;
    double acc = 0.0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < pairs;
         i += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t smp;
        const PairIdx p = pair_of(i, n, tq, smp);
        double2 *pb = psi + (smp << n), *lb = lam + (smp << n);
        double2 a = pb[p.i0], b = pb[p.i1], la = lb[p.i0], lbv = lb[p.i1];
        if (kind == 0) {
            pair_apply_d(axis, c, -s, a, b); // psi_in = u^dag psi_out
            double2 wa = a, wb = b;
            pair_apply_d(axis, dc, ds, wa, wb); // du psi_in
            acc += la.x * wa.x + la.y * wa.y + lbv.x * wb.x + lbv.y * wb.y;
            pair_apply_d(axis, c, -s, la, lbv);
        } else if (kind == 1) {
            if ((p.i1 >> q0) & 1ull) {
                b = make_double2(-b.x, -b.y);
                lbv = make_double2(-lbv.x, -lbv.y);
            }
        } else if ((p.i0 >> q0) & 1ull) {
            double2 t = a;
            a = b;
            b = t;
            t = la;
            la = lbv;
            lbv = t;
        }
        pb[p.i0] = a;
        pb[p.i1] = b;
        lb[p.i0] = la;
        lb[p.i1] = lbv;
    }
    if (kind == 0) {
        const double t = block_sum(acc);
        if (threadIdx.x == 0) gpart[blockIdx.x] = t;
    }
}

// lambda_x = 2 phase(t) psi_t, t = x ^ X; E_s = sum_x Re(conj(psi_x) phase(t) psi_t)
// (pauli_phase engine.cpp:346-372: sign from the Z parity of t, times i^y).
__global__ void __launch_bounds__(256) seed_c128(int n, uint64_t X, uint64_t Z, uint32_t y,
                                                 const double2 *psi, double2 *lam, uint32_t chunks,
                                                 double *epart) {
    const uint64_t dim = 1ull << n, per = dim / chunks;
    const uint32_t s = blockIdx.x / chunks, chunk = blockIdx.x % chunks;
    const double2 *ps = psi + s * dim;
    double2 *ls = lam + s * dim;
    double e = 0.0;
    for (uint64_t k = threadIdx.x; k < per; k += blockDim.x) {
        const uint64_t x = chunk * per + k, t = x ^ X;
        double re = ps[t].x, im = ps[t].y;
        if (__popcll(t & Z) & 1) {
            re = -re;
            im = -im;
        }
        double r2 = re, i2 = im;
        switch (y & 3u) {
        case 1: r2 = -im; i2 = re; break;
        case 2: r2 = -re; i2 = -im; break;
        case 3: r2 = im; i2 = -re; break;
        default: break;
        }
        e += ps[x].x * r2 + ps[x].y * i2;
        ls[x] = make_double2(2.0 * r2, 2.0 * i2);
    }
    const double t = block_sum(e);
    if (threadIdx.x == 0) epart[blockIdx.x] = t;
}

__global__ void c128_reduce(const double *gpart, int gblocks, const uint32_t *params, int n_rot,
                            double *grad, const double *epart, uint32_t chunks, uint32_t batch,
                            double *expect, double *loss) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n_rot) {
        double s = 0.0;
        for (int b = 0; b < gblocks; ++b) s += gpart[size_t(r) * gblocks + b];
        grad[params[r]] = s;
    }
    if (r == 0) { // per-sample expectations in chunk order, loss in sample order (engine.cpp:733-738)
        double l = 0.0;
        for (uint32_t s = 0; s < batch; ++s) {
            double e = 0.0;
            for (uint32_t c = 0; c < chunks; ++c) e += epart[size_t(s) * chunks + c];
            if (expect) expect[s] = e;
            l += e;
        }
        *loss = l;
    }
}

int grid_c128(uint64_t pairs) {
    uint64_t b = (pairs + 255) / 256;
    if (b > 148 * 8) b = 148 * 8;
    return int(b ? b : 1);
}

} // namespace

int c128_gate_grid(uint64_t pairs) { return grid_c128(pairs); }

cudaError_t launch_gate_fwd_c128(cudaStream_t st, double2 *psi, int n, uint32_t batch, int kind,
                                 int axis, uint32_t q0, uint32_t q1, const double *theta,
                                 uint32_t param) {
    const uint64_t pairs = (uint64_t(batch) << n) / 2;
    gate_fwd_c128<<<grid_c128(pairs), 256, 0, st>>>(psi, n, pairs, kind, axis, q0, q1, theta, param);
    return cudaGetLastError();
}

cudaError_t launch_gate_bwd_c128(cudaStream_t st, double2 *psi, double2 *lam, int n, uint32_t batch,
                                 int kind, int axis, uint32_t q0, uint32_t q1, const double *theta,
                                 uint32_t param, double *gpart) {
    const uint64_t pairs = (uint64_t(batch) << n) / 2;
    gate_bwd_c128<<<grid_c128(pairs), 256, 0, st>>>(psi, lam, n, pairs, kind, axis, q0, q1, theta,
                                                    param, gpart);
    return cudaGetLastError();
}

cudaError_t launch_seed_c128(cudaStream_t st, int n, uint32_t batch, uint64_t x_mask, uint64_t z_mask,
                             uint32_t y_count, const double2 *psi, double2 *lam, uint32_t chunks,
                             double *epart) {
    seed_c128<<<batch * chunks, 256, 0, st>>>(n, x_mask, z_mask, y_count, psi, lam, chunks, epart);
    return cudaGetLastError();
}

cudaError_t launch_reduce_c128(cudaStream_t st, const double *gpart, int gblocks,
                               const uint32_t *params, int n_rot, double *grad, const double *epart,
                               uint32_t chunks, uint32_t batch, double *expect, double *loss) {
    const int threads = n_rot > 1 ? n_rot : 1;
    c128_reduce<<<(threads + 127) / 128, 128, 0, st>>>(gpart, gblocks, params, n_rot, grad, epart,
                                                       chunks, batch, expect, loss);
    return cudaGetLastError();
}

} // namespace qfb
