/* TEST INFRASTRUCTURE ONLY — the CPU oracle for parity checks.
 *
 * A plain-C restatement (double precision, gate by gate) of the reference
 * qfuse algorithm for the hot path: state generation, HEA construction,
 * Pauli parsing, the circuit forward, expectation, adjoint seed and the
 * adjoint gradient. Every function cites the reference file:line it follows
 * (paths under /root/reference/proj/). Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline/reference legs may load this; the product
 * library never links it.
 *
 * Parity is pinned (see tests/test_oracle.py): against the survey's golden
 * values and against fixtures produced by the unmodified
 * reference compiled into oracle/_ref (tests/golden/make_golden.py).
 */
#ifndef QF_ORACLE_H
#define QF_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same layout as qf_gate (include/qfuse_b200.h). kind: 0 rotation, 1 CZ,
 * 2 CNOT. axis: 0 X, 1 Y, 2 Z. */
typedef struct {
    uint8_t kind;
    uint8_t axis;
    uint16_t pad;
    uint32_t q0;
    uint32_t q1;
    uint32_t param;
} qfo_gate;

uint64_t qfo_splitmix_next(uint64_t *state);
void qfo_random_state(uint32_t n_qubits, uint32_t batch, uint64_t seed, double *out);
void qfo_random_parameters(uint64_t count, uint64_t seed, double *out);
int qfo_build_hea(uint32_t n_qubits, uint32_t layers, qfo_gate *out, uint64_t cap,
                  uint64_t *n_gates, uint32_t *n_params);
void qfo_repeated_ixyz(uint32_t n_qubits, char *out /* n+1 bytes */);
int qfo_parse_pauli(const char *label, uint32_t expected_n, uint64_t *x_mask,
                    uint64_t *z_mask, uint32_t *y_count);

int qfo_forward(const qfo_gate *gates, uint64_t n_gates, uint32_t n_qubits,
                double *psi /* in/out, batch * 2^(n+1) */, uint32_t batch,
                const double *theta);
void qfo_expectation(const double *psi, uint32_t n_qubits, uint32_t batch, uint64_t x_mask,
                     uint64_t z_mask, uint32_t y_count, double *out /* batch */);
void qfo_seed_adjoint(const double *psi, double *lambda, uint32_t n_qubits, uint32_t batch,
                      uint64_t x_mask, uint64_t z_mask, uint32_t y_count);
int qfo_gradient(const qfo_gate *gates, uint64_t n_gates, uint32_t n_qubits,
                 uint32_t n_params, const double *psi0, uint32_t batch, const double *theta,
                 uint64_t x_mask, uint64_t z_mask, uint32_t y_count, double *loss,
                 double *grad /* n_params, summed over batch */,
                 double *expect /* batch, nullable */);
int qfo_gradient_f32in(const qfo_gate *gates, uint64_t n_gates, uint32_t n_qubits,
                       uint32_t n_params, const float *psi0, uint32_t batch,
                       const double *theta, uint64_t x_mask, uint64_t z_mask,
                       uint32_t y_count, double *loss, double *grad, double *expect);

#ifdef __cplusplus
}
#endif

#endif
