// Per-call theta preparation, reductions and the synthetic input generator.
//
//   prep_sections_kernel: compose each single-qubit run in fp64 (circuit.cpp:61-87,
//       fusion.cpp:127-152 order) and split it U = e^{id} Rz(a) Ry(b) Rz(g).
//   diag_tables_kernel:   per-stage diagonal tables.
//   reduce/finalize:      fixed-order fp64 reductions; gradient of every
//       reference rotation from K (grad = Re Tr(dg K g^dag), the block backward of
//       engine.cpp:265-342 written on the 2x2 cross correlation).
//   rand_*:               new_random_state (statevec.cpp:32-53) on the device.
#include "qf_device.cuh"

namespace qfb {
namespace {

// --------------------------------------------------- per-call θ prep
__device__ inline double2 zmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ inline double2 zconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ inline double2 zadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

struct M2 {
    double2 a, b, c, d; // [[a, b], [c, d]]
};
__device__ inline M2 mmul(const M2 &x, const M2 &y) {
    return {zadd(zmul(x.a, y.a), zmul(x.b, y.c)), zadd(zmul(x.a, y.b), zmul(x.b, y.d)),
            zadd(zmul(x.c, y.a), zmul(x.d, y.c)), zadd(zmul(x.c, y.b), zmul(x.d, y.d))};
}
__device__ inline M2 mdag(const M2 &x) { return {zconj(x.a), zconj(x.c), zconj(x.b), zconj(x.d)}; }
// rotation_matrix / rotation_derivative, circuit.cpp:61-87.
__device__ inline M2 rot_m(int axis, double theta, bool deriv) {
    double s, c;
    sincos(theta / 2.0, &s, &c);
    double a = c, b = s;
    if (deriv) {
        a = -0.5 * s;
        b = 0.5 * c;
    }
    switch (axis) {
    case 0: return {{a, 0}, {0, -b}, {0, -b}, {a, 0}};
    case 1: return {{a, 0}, {-b, 0}, {b, 0}, {a, 0}};
    default: return {{a, -b}, {0, 0}, {0, 0}, {a, b}};
    }
}
__device__ inline M2 hadamard() {
    const double r = 0.70710678118654752440;
    return {{r, 0}, {r, 0}, {r, 0}, {-r, 0}};
}
__device__ inline M2 sec_gate(uint32_t enc, const double *theta, bool deriv) {
    const uint32_t kind = enc & 3u;
    if (kind == kSecH) return hadamard();
    return rot_m(int(kind), theta[enc >> 2], deriv);
}

// One thread per section: compose the run's 2x2 in fp64, decompose
// U = e^{i delta} Rz(alpha) Ry(beta) Rz(gamma) and scatter the stage data.
__global__ void prep_sections_kernel(int n_sec, const uint32_t *sec_q, const uint32_t *sec_stage,
                                     const uint32_t *sec_alpha_row, const uint32_t *sec_off,
                                     const uint32_t *sec_gates, const double *theta, int n,
                                     float2 *ry, double *wg, double *wa, double *sec_gamma,
                                     double *sec_phase) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_sec) return;
    M2 u{{1, 0}, {0, 0}, {0, 0}, {1, 0}};
    for (uint32_t k = sec_off[i]; k < sec_off[i + 1]; ++k) u = mmul(sec_gate(sec_gates[k], theta, false), u);
    // normalise to SU(2): v = u / sqrt(det u)
    const double2 det = zadd(zmul(u.a, u.d), make_double2(-(u.b.x * u.c.x - u.b.y * u.c.y),
                                                          -(u.b.x * u.c.y + u.b.y * u.c.x)));
    const double dr = sqrt(hypot(det.x, det.y)), dth = 0.5 * atan2(det.y, det.x);
    const double2 inv = make_double2(cos(dth) / dr, -sin(dth) / dr);
    const double2 a = zmul(u.a, inv), b = zmul(u.c, inv);
    const double ca = hypot(a.x, a.y), cb = hypot(b.x, b.y);
    const double beta = 2.0 * atan2(cb, ca);
    double alpha, gamma;
    if (cb < 1e-13) {
        alpha = 0.0;
        gamma = -2.0 * atan2(a.y, a.x);
    } else if (ca < 1e-13) {
        alpha = 2.0 * atan2(b.y, b.x);
        gamma = 0.0;
    } else {
        const double ga = atan2(a.y, a.x), gb = atan2(b.y, b.x);
        alpha = gb - ga;
        gamma = -ga - gb;
    }
    const uint32_t q = sec_q[i], st = sec_stage[i];
    double sb, cbt;
    sincos(0.5 * beta, &sb, &cbt);
    ry[size_t(st) * n + q] = make_float2(float(cbt), float(sb));
    wg[size_t(st) * n + q] = gamma;
    wa[size_t(sec_alpha_row[i]) * n + q] = alpha;
    sec_gamma[i] = gamma;
    // global phase the device model drops: U = e^{i dth} Rz(a) Ry(b) Rz(g) and the
    // diagonal tables apply Rz(w) as diag(1, e^{i w}) = e^{i w / 2} Rz(w)
    sec_phase[i] = dth - 0.5 * (alpha + gamma);
}

// Forward-state readout only: wfinal[n] = sum of the sections' dropped phases
// (fixed order: strided per-thread sums, then a sequential sum over threads).
__global__ void phase_sum_kernel(int n_sec, const double *sec_phase, int n, double *wfinal) {
    __shared__ double part[256];
    double s = 0.0;
    for (int i = threadIdx.x; i < n_sec; i += blockDim.x) s += sec_phase[i];
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < int(blockDim.x); ++k) t += part[k];
        wfinal[n] = t;
    }
}

// Per stage: e^{i sum_q w_q x_q} tables of D_s in the layout of the pass that
// applies it (fp64 -> complex64). dq[layout][0..27] = qubit of register bit
// 0..3, thread bit 0..7, tile bit 0..15 (-1: none / sample bit).
__global__ void diag_tables_kernel(int stages, int n, const double *wg, const double *wa,
                                   const int *stage_layout, const int *dq, DiagTab *dt,
                                   double *wfinal) {
    const int s = blockIdx.x;
    if (s == stages) {
        for (int q = threadIdx.x; q < n; q += blockDim.x)
            wfinal[q] = wg[size_t(stages) * n + q] + wa[size_t(stages) * n + q];
        return;
    }
    const int *m = dq + stage_layout[s] * 28;
    for (int e = threadIdx.x; e < 16 + 3 * 256; e += blockDim.x) {
        int base, bits, idx;
        float2 *dst;
        if (e < 16) { base = 0; bits = 4; idx = e; dst = dt[s].treg + idx; }
        else if (e < 272) { base = 4; bits = 8; idx = e - 16; dst = dt[s].tthr + idx; }
        else if (e < 528) { base = 12; bits = 8; idx = e - 272; dst = dt[s].tt1 + idx; }
        else { base = 20; bits = 8; idx = e - 528; dst = dt[s].tt2 + idx; }
        double ang = 0.0;
        for (int b = 0; b < bits; ++b) {
            const int q = m[base + b];
            if (q >= 0 && q < n && ((idx >> b) & 1)) ang += wg[size_t(s) * n + q] + wa[size_t(s) * n + q];
        }
        double sn, cs;
        sincos(ang, &sn, &cs);
        *dst = make_float2(float(cs), float(sn));
    }
}

// Wide-group register/thread tables (qf_pass_wide.cu) of the stages layout 0 applies.
__global__ void diag_tables_wide_kernel(int n, const double *wg, const double *wa,
                                        const int *stage_layout, const int *dqw, DiagTabW *dtw) {
    const int s = blockIdx.x;
    if (stage_layout[s] != 0) return;
    const int e = threadIdx.x; // 0..63 register entries, 64..127 thread entries
    const int base = e < 64 ? 0 : 6, idx = e & 63;
    double ang = 0.0;
    for (int b = 0; b < 6; ++b) {
        const int q = dqw[base + b];
        if (q >= 0 && q < n && ((idx >> b) & 1)) ang += wg[size_t(s) * n + q] + wa[size_t(s) * n + q];
    }
    double sn, cs;
    sincos(ang, &sn, &cs);
    (e < 64 ? dtw[s].treg : dtw[s].tthr)[idx] = make_float2(float(cs), float(sn));
}

// kout[e] = sum over CTAs (fixed order) of kpart[cta][e]; expect[s] = sum of
// the seed kernel's chunk partials.
__global__ void reduce_kernel(long long entries, int grid, const double *kpart, double *kout,
                              const double *epart, int chunks, uint32_t batch, double *expect) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < entries) {
        double s = 0.0;
        for (int g = 0; g < grid; ++g) s += kpart[size_t(g) * entries + i];
        kout[i] = s;
    }
    if (epart && i < batch) {
        double s = 0.0;
        for (int c = 0; c < chunks; ++c) s += epart[size_t(i) * chunks + c];
        expect[i] = s;
    }
}

// loss = sum_s E_s (engine.cpp:733-738), fixed-order warp reduction.
__global__ void loss_kernel(const double *expect, uint32_t batch, double *loss) {
    double s = 0.0;
    for (uint32_t i = threadIdx.x; i < batch; i += 32) s += expect[i];
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
    if (threadIdx.x == 0) *loss = s;
}

// One thread per section: K at the point before Ry(beta) -> K at the run
// start (Rz(gamma)^dag), then walk the run's gates: grad = Re Tr(dg K g^dag),
// K <- g K g^dag. Only the traceless anti-Hermitian part of K (X, Y, Z from
// the pass kernels) enters Re Tr(dg K g^dag), so K is rebuilt from it.
__global__ void finalize_kernel(int n_sec, const uint32_t *sec_q, const uint32_t *sec_stage,
                                const uint32_t *sec_off, const uint32_t *sec_gates,
                                const double *sec_gamma, const double *theta, int n,
                                const double *kout, double *grad, const double *loss) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_sec) return;
    const double *k = kout + (size_t(sec_stage[i]) * n + sec_q[i]) * 8;
    const double g = sec_gamma[i];
    const double2 e = make_double2(cos(g), sin(g));
    // K~ = (i/2)(X sx + Y sy + Z sz) carries exactly the Im Tr(sigma_m K) the
    // gradients depend on (qf_device.cuh kbit3): [[iZ, Y + iX], [-Y + iX, -iZ]] / 2.
    const double X = k[0], Y = k[1], Z = k[2];
    (void)loss;
    M2 K{{0.0, 0.5 * Z}, zmul(make_double2(0.5 * Y, 0.5 * X), e),
         zmul(make_double2(-0.5 * Y, 0.5 * X), zconj(e)), {0.0, -0.5 * Z}};
    for (uint32_t j = sec_off[i]; j < sec_off[i + 1]; ++j) {
        const uint32_t enc = sec_gates[j];
        const M2 gm = sec_gate(enc, theta, false);
        if ((enc & 3u) != kSecH) {
            const M2 dg = sec_gate(enc, theta, true);
            const M2 t = mmul(mmul(dg, K), mdag(gm));
            grad[enc >> 2] = t.a.x + t.d.x;
        }
        K = mmul(mmul(gm, K), mdag(gm));
    }
}

// Z(s) = cos(b) Z(s-1) - sin(b) X(s-1), b = beta_{s-1}(q): Z commutes with every
// diagonal and every other qubit's gate between Ry_{s-1}(q) and Ry_s(q), and
// Ry(b)^dag sz Ry(b) = cos(b) sz - sin(b) sx. One thread per qubit, in stage order.
__global__ void zchain_kernel(int stages, int n, const float2 *__restrict__ ry,
                              double *__restrict__ kout) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    double z = kout[size_t(q) * 8 + 2]; // stage 0: measured
#pragma unroll 8
    for (int s = 1; s < stages; ++s) {
        const float2 cs = __ldg(&ry[size_t(s - 1) * n + q]);
        const double x = kout[(size_t(s - 1) * n + q) * 8];
        const double c = cs.x, sn = cs.y;
        z = (c * c - sn * sn) * z - (2.0 * c * sn) * x;
        kout[(size_t(s) * n + q) * 8 + 2] = z;
    }
}

__device__ __forceinline__ uint64_t sm_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double2 bm_amp(uint64_t seed, uint64_t a) {
    const uint64_t j = 2 * a; // draws j (u1) and j+1 (u2)
    const uint64_t z0 = sm_mix(seed + (j + 1) * 0x9e3779b97f4a7c15ull);
    const uint64_t z1 = sm_mix(seed + (j + 2) * 0x9e3779b97f4a7c15ull);
    const double u1 = double((z0 >> 11) + 1) * 0x1.0p-53;
    const double u2 = double(z1 >> 11) * 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u1));
    double s, c;
    sincos(2.0 * 3.14159265358979323846 * u2, &s, &c);
    return make_double2(r * c, r * s);
}
__global__ void rand_norm_kernel(uint64_t seed, uint64_t first, int n, uint32_t chunks,
                                 double *part) {
    const uint64_t dim = 1ull << n, per = dim / chunks;
    const uint32_t s = blockIdx.x / chunks, c = blockIdx.x % chunks;
    double acc = 0.0;
    for (uint64_t k = threadIdx.x; k < per; k += blockDim.x) {
        const double2 v = bm_amp(seed, (first + s) * dim + c * per + k);
        acc += v.x * v.x + v.y * v.y;
    }
    __shared__ double red[8];
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0;
        for (int w = 0; w < 8; ++w) t += red[w];
        part[blockIdx.x] = t;
    }
}
__global__ void rand_write_kernel(uint64_t seed, uint64_t first, int n, uint32_t chunks,
                                  const double *part, float2 *out) {
    const uint64_t dim = 1ull << n, per = dim / chunks;
    const uint32_t s = blockIdx.x / chunks, c = blockIdx.x % chunks;
    double nrm = 0.0;
    for (uint32_t i = 0; i < chunks; ++i) nrm += part[size_t(s) * chunks + i];
    const double inv = 1.0 / sqrt(nrm);
    for (uint64_t k = threadIdx.x; k < per; k += blockDim.x) {
        const uint64_t x = c * per + k;
        const double2 v = bm_amp(seed, (first + s) * dim + x);
        out[s * dim + x] = make_float2(float(v.x * inv), float(v.y * inv));
    }
}
} // namespace

cudaError_t launch_prep_sections(cudaStream_t st, int n_sec, const uint32_t *sec_q,
                                 const uint32_t *sec_stage, const uint32_t *sec_alpha_row,
                                 const uint32_t *sec_off, const uint32_t *sec_gates,
                                 const double *theta, int n, float2 *ry, double *wg, double *wa,
                                 double *sec_gamma, double *sec_phase) {
    if (n_sec == 0) return cudaSuccess;
    prep_sections_kernel<<<(n_sec + 127) / 128, 128, 0, st>>>(
        n_sec, sec_q, sec_stage, sec_alpha_row, sec_off, sec_gates, theta, n, ry, wg, wa, sec_gamma,
        sec_phase);
    return cudaGetLastError();
}

cudaError_t launch_phase_sum(cudaStream_t st, int n_sec, const double *sec_phase, int n,
                             double *wfinal) {
    phase_sum_kernel<<<1, 256, 0, st>>>(n_sec, sec_phase, n, wfinal);
    return cudaGetLastError();
}

cudaError_t launch_diag_tables(cudaStream_t st, int stages, int n, const double *wg,
                               const double *wa, const int *stage_layout, const int *dq,
                               DiagTab *dt, double *wfinal) {
    diag_tables_kernel<<<stages + 1, 256, 0, st>>>(stages, n, wg, wa, stage_layout, dq, dt, wfinal);
    return cudaGetLastError();
}

cudaError_t launch_diag_tables_wide(cudaStream_t st, int stages, int n, const double *wg,
                                    const double *wa, const int *stage_layout, const int *dqw,
                                    DiagTabW *dtw) {
    if (stages == 0) return cudaSuccess;
    diag_tables_wide_kernel<<<stages, 128, 0, st>>>(n, wg, wa, stage_layout, dqw, dtw);
    return cudaGetLastError();
}

cudaError_t launch_reduce(cudaStream_t st, long long entries, int grid, const double *kpart,
                          double *kout, const double *epart, int chunks, uint32_t batch,
                          double *expect) {
    const long long work = entries > (long long)batch ? entries : (long long)batch;
    if (work == 0) return cudaSuccess;
    reduce_kernel<<<unsigned((work + 255) / 256), 256, 0, st>>>(entries, grid, kpart, kout, epart,
                                                                chunks, batch, expect);
    return cudaGetLastError();
}

cudaError_t launch_finalize(cudaStream_t st, int n_sec, const uint32_t *sec_q,
                            const uint32_t *sec_stage, const uint32_t *sec_off,
                            const uint32_t *sec_gates, const double *sec_gamma,
                            const double *theta, int n, const double *kout, double *grad,
                            const double *expect, uint32_t batch, double *loss) {
    loss_kernel<<<1, 32, 0, st>>>(expect, batch, loss);
    if (n_sec > 0)
        finalize_kernel<<<(n_sec + 127) / 128, 128, 0, st>>>(n_sec, sec_q, sec_stage, sec_off,
                                                             sec_gates, sec_gamma, theta, n, kout,
                                                             grad, loss);
    return cudaGetLastError();
}

cudaError_t launch_zchain(cudaStream_t st, int stages, int n, const float2 *ry, double *kout) {
    if (stages <= 1 || n <= 0) return cudaSuccess;
    zchain_kernel<<<1, 32, 0, st>>>(stages, n, ry, kout);
    return cudaGetLastError();
}

cudaError_t launch_random_state(cudaStream_t st, uint64_t seed, uint64_t first_sample, int n,
                                uint32_t batch, double *scratch /* batch*chunks */,
                                float2 *out) {
    const uint64_t dim = 1ull << n;
    const uint32_t chunks = dim >= 4096 ? uint32_t(dim / 4096) : 1u;
    rand_norm_kernel<<<batch * chunks, 256, 0, st>>>(seed, first_sample, n, chunks, scratch);
    rand_write_kernel<<<batch * chunks, 256, 0, st>>>(seed, first_sample, n, chunks, scratch, out);
    return cudaGetLastError();
}
} // namespace qfb
