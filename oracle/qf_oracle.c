/* TEST INFRASTRUCTURE ONLY — see qf_oracle.h.
 *
 * Double-precision, one-gate-at-a-time restatement of the reference
 * algorithm. References are to /root/reference/proj/.
 */
#include "qf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define QFO_PI 3.14159265358979323846

/* SplitMix64 step — include/qfuse/bits.hpp:44-49. */
uint64_t qfo_splitmix_next(uint64_t *state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

/* next_unit (bits.hpp:52) and next_unit_open (bits.hpp:55-57). */
static double unit(uint64_t *st) { return (double)(qfo_splitmix_next(st) >> 11) * 0x1.0p-53; }
static double unit_open(uint64_t *st) {
    return (double)((qfo_splitmix_next(st) >> 11) + 1) * 0x1.0p-53;
}

/* new_random_state — statevec.cpp:32-53: one stream for the whole batch,
 * samples in order, two draws (Box-Muller, bits.hpp:61-67) per amplitude,
 * per-sample normalisation in double. */
void qfo_random_state(uint32_t n, uint32_t batch, uint64_t seed, double *out) {
    uint64_t st = seed;
    const uint64_t dim = 1ull << n;
    for (uint32_t s = 0; s < batch; ++s) {
        double *p = out + (size_t)s * 2 * dim;
        double norm_sq = 0.0;
        for (uint64_t x = 0; x < dim; ++x) {
            const double u1 = unit_open(&st);
            const double u2 = unit(&st);
            const double r = sqrt(-2.0 * log(u1));
            const double t = 2.0 * QFO_PI * u2;
            p[2 * x] = r * cos(t);
            p[2 * x + 1] = r * sin(t);
            norm_sq += p[2 * x] * p[2 * x] + p[2 * x + 1] * p[2 * x + 1];
        }
        const double inv = 1.0 / sqrt(norm_sq);
        for (uint64_t i = 0; i < 2 * dim; ++i) p[i] *= inv;
    }
}

/* random_parameters — circuit.cpp:214-221. */
void qfo_random_parameters(uint64_t count, uint64_t seed, double *out) {
    uint64_t st = seed;
    for (uint64_t i = 0; i < count; ++i) out[i] = unit(&st) * 2.0 * QFO_PI;
}

/* build_hea — circuit.cpp:89-114: per layer Rx,Ry,Rz on each qubit in
 * order, then the CZ ring (q, q+1 mod n); n = 2 uses one CZ. */
int qfo_build_hea(uint32_t n, uint32_t layers, qfo_gate *out, uint64_t cap,
                  uint64_t *n_gates, uint32_t *n_params) {
    if (n < 2 || layers == 0) return 2;
    const uint32_t ents = n == 2 ? 1 : n;
    const uint64_t total = (uint64_t)layers * (3ull * n + ents);
    *n_gates = total;
    *n_params = 3u * n * layers;
    uint64_t g = 0;
    uint32_t param = 0;
    for (uint32_t l = 0; l < layers; ++l) {
        for (uint32_t q = 0; q < n; ++q) {
            for (uint8_t a = 0; a < 3; ++a) {
                if (g < cap) {
                    qfo_gate gt = {0, a, 0, q, 0, param};
                    out[g] = gt;
                }
                ++g;
                ++param;
            }
        }
        for (uint32_t q = 0; q < ents; ++q) {
            if (g < cap) {
                qfo_gate gt = {1, 0, 0, q, (q + 1) % n, 0};
                out[g] = gt;
            }
            ++g;
        }
    }
    return 0;
}

/* repeated_ixyz_label — circuit.cpp:205-212. */
void qfo_repeated_ixyz(uint32_t n, char *out) {
    static const char cyc[4] = {'I', 'X', 'Y', 'Z'};
    for (uint32_t i = 0; i < n; ++i) out[i] = cyc[i % 4];
    out[n] = '\0';
}

/* parse_pauli — circuit.cpp:158-192 (leftmost char acts on qubit n-1),
 * y_count = popcount(x & z) (circuit.cpp:155). */
int qfo_parse_pauli(const char *label, uint32_t expected_n, uint64_t *x_mask,
                    uint64_t *z_mask, uint32_t *y_count) {
    const size_t n = strlen(label);
    if (n == 0 || n > 64) return 2;
    if (expected_n != 0 && n != expected_n) return 2;
    uint64_t x = 0, z = 0;
    for (size_t i = 0; i < n; ++i) {
        const uint64_t bit = 1ull << (n - 1 - i);
        switch (label[i]) {
        case 'I': break;
        case 'X': x |= bit; break;
        case 'Y': x |= bit; z |= bit; break;
        case 'Z': z |= bit; break;
        default: return 2;
        }
    }
    *x_mask = x;
    *z_mask = z;
    *y_count = (uint32_t)__builtin_popcountll(x & z);
    return 0;
}

/* u = cI - i s P on the pair (a, b) — engine.cpp:36-59 (same form for u^dag
 * with s -> -s and for du/dtheta with (c, s) -> (-s/2, c/2)). */
static void pair_apply(int axis, double c, double s, double *ar, double *ai, double *br,
                       double *bi) {
    const double a_re = *ar, a_im = *ai, b_re = *br, b_im = *bi;
    switch (axis) {
    case 0:
        *ar = c * a_re + s * b_im;
        *ai = c * a_im - s * b_re;
        *br = c * b_re + s * a_im;
        *bi = c * b_im - s * a_re;
        break;
    case 1:
        *ar = c * a_re - s * b_re;
        *ai = c * a_im - s * b_im;
        *br = s * a_re + c * b_re;
        *bi = s * a_im + c * b_im;
        break;
    default:
        *ar = c * a_re + s * a_im;
        *ai = c * a_im - s * a_re;
        *br = c * b_re - s * b_im;
        *bi = c * b_im + s * b_re;
        break;
    }
}

/* Rotation on one sample — apply_rotation_kernel, engine.cpp:172-202. */
static void rot_sample(double *p, uint32_t n, int axis, double c, double s, uint32_t t) {
    const uint64_t pairs = 1ull << (n - 1), mask = 1ull << t, lo = mask - 1;
    for (uint64_t k = 0; k < pairs; ++k) {
        const uint64_t i0 = ((k & ~lo) << 1) | (k & lo), i1 = i0 | mask; /* bits.hpp:26-28 */
        pair_apply(axis, c, s, &p[2 * i0], &p[2 * i0 + 1], &p[2 * i1], &p[2 * i1 + 1]);
    }
}

/* CZ sign flip — apply_cz_kernel, engine.cpp:111-136 (one mask). */
static void cz_sample(double *p, uint32_t n, uint32_t a, uint32_t b) {
    const uint64_t dim = 1ull << n, m = (1ull << a) | (1ull << b);
    for (uint64_t x = 0; x < dim; ++x)
        if ((x & m) == m) { p[2 * x] = -p[2 * x]; p[2 * x + 1] = -p[2 * x + 1]; }
}

/* CNOT permutation — apply_cnot_kernel, engine.cpp:142-170 (self-inverse). */
static void cnot_sample(double *p, uint32_t n, uint32_t c, uint32_t t) {
    const uint64_t dim = 1ull << n, cm = 1ull << c, tm = 1ull << t;
    for (uint64_t x = 0; x < dim; ++x) {
        if ((x & cm) && !(x & tm)) {
            const uint64_t y = x | tm;
            double r = p[2 * x], i = p[2 * x + 1];
            p[2 * x] = p[2 * y]; p[2 * x + 1] = p[2 * y + 1];
            p[2 * y] = r; p[2 * y + 1] = i;
        }
    }
}

static int check_gates(const qfo_gate *g, uint64_t ng, uint32_t n) {
    for (uint64_t i = 0; i < ng; ++i) {
        if (g[i].q0 >= n || g[i].kind > 2 || g[i].axis > 2) return 2;
        if (g[i].kind != 0 && (g[i].q1 >= n || g[i].q1 == g[i].q0)) return 2;
    }
    return 0;
}

static void forward_sample(const qfo_gate *gates, uint64_t ng, uint32_t n, double *p,
                           const double *theta) {
    for (uint64_t i = 0; i < ng; ++i) {
        const qfo_gate *g = &gates[i];
        if (g->kind == 0) {
            const double h = theta[g->param] / 2.0;
            rot_sample(p, n, g->axis, cos(h), sin(h), g->q0);
        } else if (g->kind == 1) {
            cz_sample(p, n, g->q0, g->q1);
        } else {
            cnot_sample(p, n, g->q0, g->q1);
        }
    }
}

/* Gate-by-gate forward — naive_forward_range, engine.cpp:757-800. */
int qfo_forward(const qfo_gate *gates, uint64_t ng, uint32_t n, double *psi, uint32_t batch,
                const double *theta) {
    if (check_gates(gates, ng, n)) return 2;
    const size_t stride = (size_t)2 << n;
    for (uint32_t s = 0; s < batch; ++s) forward_sample(gates, ng, n, psi + s * stride, theta);
    return 0;
}

/* Phase of <x|O|x^X>: Z-mask parity of the source index times i^y_count —
 * pauli_phase, engine.cpp:346-372. */
static void pauli_phase(uint64_t target, uint64_t z_mask, uint32_t y_count, double *re,
                        double *im) {
    if (__builtin_popcountll(target & z_mask) & 1) { *re = -*re; *im = -*im; }
    double t;
    switch (y_count & 3) {
    case 1: t = *re; *re = -*im; *im = t; break;
    case 2: *re = -*re; *im = -*im; break;
    case 3: t = *re; *re = *im; *im = -t; break;
    default: break;
    }
}

/* expectation_kernel — engine.cpp:374-409 (sum in index order, double). */
void qfo_expectation(const double *psi, uint32_t n, uint32_t batch, uint64_t x_mask,
                     uint64_t z_mask, uint32_t y_count, double *out) {
    const uint64_t dim = 1ull << n;
    const size_t stride = (size_t)2 << n;
    for (uint32_t s = 0; s < batch; ++s) {
        const double *p = psi + s * stride;
        double acc = 0.0;
        for (uint64_t x = 0; x < dim; ++x) {
            const uint64_t t = x ^ x_mask;
            double kr = p[2 * t], ki = p[2 * t + 1];
            pauli_phase(t, z_mask, y_count, &kr, &ki);
            acc += p[2 * x] * kr + p[2 * x + 1] * ki;
        }
        out[s] = acc;
    }
}

/* seed_adjoint_kernel — engine.cpp:411-435: lambda = 2 O psi. */
void qfo_seed_adjoint(const double *psi, double *lam, uint32_t n, uint32_t batch,
                      uint64_t x_mask, uint64_t z_mask, uint32_t y_count) {
    const uint64_t dim = 1ull << n;
    const size_t stride = (size_t)2 << n;
    for (uint32_t s = 0; s < batch; ++s) {
        const double *p = psi + s * stride;
        double *l = lam + s * stride;
        for (uint64_t x = 0; x < dim; ++x) {
            const uint64_t t = x ^ x_mask;
            double kr = p[2 * t], ki = p[2 * t + 1];
            pauli_phase(t, z_mask, y_count, &kr, &ki);
            l[2 * x] = 2.0 * kr;
            l[2 * x + 1] = 2.0 * ki;
        }
    }
}

/* Adjoint gradient — naive_gradient (engine.cpp:856-894) with the per-gate
 * backward of rotation_backward_kernel (engine.cpp:207-256): for each
 * rotation, walking the gates in reverse, accumulate Re[lambda^dag du psi_in]
 * and advance lambda <- u^dag lambda. The reference reads psi_in from a
 * ledger of stored gate inputs (engine.cpp:767,815-822); in double precision
 * this restatement recovers it exactly enough (<1e-14) by applying u^dag to
 * the running state, which keeps memory O(state) for deep circuits. CZ and
 * CNOT are involutions applied to both vectors (engine.cpp:833-848). */
static void gradient_sample(const qfo_gate *gates, uint64_t ng, uint32_t n,
                            const double *psi0, const double *theta, uint64_t x_mask,
                            uint64_t z_mask, uint32_t y_count, double *grad, double *e_out,
                            double *psi, double *lam) {
    const uint64_t dim = 1ull << n;
    memcpy(psi, psi0, sizeof(double) * 2 * dim);
    forward_sample(gates, ng, n, psi, theta);
    qfo_expectation(psi, n, 1, x_mask, z_mask, y_count, e_out);
    qfo_seed_adjoint(psi, lam, n, 1, x_mask, z_mask, y_count);
    for (uint64_t i = ng; i-- > 0;) {
        const qfo_gate *g = &gates[i];
        if (g->kind == 0) {
            const double h = theta[g->param] / 2.0, c = cos(h), s = sin(h);
            rot_sample(psi, n, g->axis, c, -s, g->q0); /* psi_in = u^dag psi_out */
            const uint64_t pairs = 1ull << (n - 1), mask = 1ull << g->q0, lo = mask - 1;
            double acc = 0.0;
            for (uint64_t k = 0; k < pairs; ++k) {
                const uint64_t i0 = ((k & ~lo) << 1) | (k & lo), i1 = i0 | mask;
                double war = psi[2 * i0], wai = psi[2 * i0 + 1];
                double wbr = psi[2 * i1], wbi = psi[2 * i1 + 1];
                pair_apply(g->axis, -0.5 * s, 0.5 * c, &war, &wai, &wbr, &wbi);
                acc += lam[2 * i0] * war + lam[2 * i0 + 1] * wai + lam[2 * i1] * wbr +
                       lam[2 * i1 + 1] * wbi;
            }
            grad[g->param] += acc;
            rot_sample(lam, n, g->axis, c, -s, g->q0);
        } else if (g->kind == 1) {
            cz_sample(psi, n, g->q0, g->q1);
            cz_sample(lam, n, g->q0, g->q1);
        } else {
            cnot_sample(psi, n, g->q0, g->q1);
            cnot_sample(lam, n, g->q0, g->q1);
        }
    }
}

int qfo_gradient(const qfo_gate *gates, uint64_t ng, uint32_t n, uint32_t n_params,
                 const double *psi0, uint32_t batch, const double *theta, uint64_t x_mask,
                 uint64_t z_mask, uint32_t y_count, double *loss, double *grad,
                 double *expect) {
    if (n == 0 || n > 30 || batch == 0) return 2;
    if (check_gates(gates, ng, n)) return 2;
    for (uint64_t i = 0; i < ng; ++i)
        if (gates[i].kind == 0 && gates[i].param >= n_params) return 2;
    const uint64_t dim = 1ull << n;
    const size_t stride = 2 * dim;
    double *per = calloc((size_t)batch * n_params + batch, sizeof(double));
    if (!per) return 3;
    double *es = per + (size_t)batch * n_params;
    int fail = 0;
#pragma omp parallel
    {
        double *psi = malloc(sizeof(double) * stride);
        double *lam = malloc(sizeof(double) * stride);
        if (!psi || !lam) {
#pragma omp atomic write
            fail = 1;
        } else {
#pragma omp for schedule(dynamic, 1)
            for (uint32_t s = 0; s < batch; ++s)
                gradient_sample(gates, ng, n, psi0 + s * stride, theta, x_mask, z_mask, y_count,
                                per + (size_t)s * n_params, &es[s], psi, lam);
        }
        free(psi);
        free(lam);
    }
    if (fail) { free(per); return 3; }
    /* loss = sum_s E_s (engine.cpp:733-738); gradients summed over samples
     * in sample order so the result is thread-count independent. */
    double l = 0.0;
    for (uint32_t j = 0; j < n_params; ++j) grad[j] = 0.0;
    for (uint32_t s = 0; s < batch; ++s) {
        l += es[s];
        for (uint32_t j = 0; j < n_params; ++j) grad[j] += per[(size_t)s * n_params + j];
        if (expect) expect[s] = es[s];
    }
    *loss = l;
    free(per);
    return 0;
}

int qfo_gradient_f32in(const qfo_gate *gates, uint64_t ng, uint32_t n, uint32_t n_params,
                       const float *psi0, uint32_t batch, const double *theta,
                       uint64_t x_mask, uint64_t z_mask, uint32_t y_count, double *loss,
                       double *grad, double *expect) {
    const size_t count = (size_t)batch << (n + 1);
    double *p = malloc(sizeof(double) * count);
    if (!p) return 3;
    for (size_t i = 0; i < count; ++i) p[i] = (double)psi0[i];
    const int rc = qfo_gradient(gates, ng, n, n_params, p, batch, theta, x_mask, z_mask,
                                y_count, loss, grad, expect);
    free(p);
    return rc;
}
