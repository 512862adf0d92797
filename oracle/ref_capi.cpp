// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the *unmodified* reference library (qfuse, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It lets
// the pytest suite, the golden-vector generator and bench.py's reference arm
// call the reference's own public C++ API:
//   qfuse::gradient<T>            engine.hpp:139-142  (engine.cpp:716-755)
//   qfuse::run_checkpointed<T>    checkpoint.hpp:65-69 (checkpoint.cpp:144-163)
//   qfuse::naive_gradient<T>      engine.hpp:146-149  (engine.cpp:856-894)
//   qfuse::forward<T>/expectation engine.cpp:704-714, :582-589
//   qfuse::oracle::parameter_shift_gradient  oracle.cpp:269-290
//   qfuse::new_random_state<T>    statevec.cpp:32-53
//   qfuse::random_parameters      circuit.cpp:214-221
//   qfuse::build_hea              circuit.cpp:89-114
//   qfuse::parse_pauli            circuit.cpp:158-192
// Only plain pointers cross this boundary; errors map to the same codes the
// product C-ABI uses (2 invalid argument, 3 capacity, 4 other).
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include <omp.h>

#include "qfuse/checkpoint.hpp"
#include "qfuse/circuit.hpp"
#include "qfuse/common.hpp"
#include "qfuse/engine.hpp"
#include "qfuse/fusion.hpp"
#include "qfuse/oracle.hpp"
#include "qfuse/statevec.hpp"

namespace {

thread_local std::string g_err;

struct RefGate { // layout identical to qf_gate in include/qfuse_b200.h
    uint8_t kind;
    uint8_t axis;
    uint16_t pad;
    uint32_t q0;
    uint32_t q1;
    uint32_t param;
};

template <class F> int guarded(F &&f) {
    try {
        f();
        return 0;
    } catch (const qfuse::CapacityError &e) {
        g_err = e.what();
        return 3;
    } catch (const std::invalid_argument &e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception &e) {
        g_err = e.what();
        return 4;
    }
}

qfuse::Circuit make_circuit(const RefGate *gates, size_t n_gates, uint32_t n_qubits,
                            uint32_t n_params) {
    std::vector<qfuse::Gate> gs;
    gs.reserve(n_gates);
    for (size_t i = 0; i < n_gates; ++i) {
        const RefGate &g = gates[i];
        const auto axis = static_cast<qfuse::Axis>(g.axis);
        switch (g.kind) {
        case 0: gs.push_back(qfuse::Gate::rotation(axis, g.q0, g.param)); break;
        case 1: gs.push_back(qfuse::Gate::cz(g.q0, g.q1)); break;
        case 2: gs.push_back(qfuse::Gate::cnot(g.q0, g.q1)); break;
        default: throw std::invalid_argument("ref_capi: unknown gate kind");
        }
    }
    return qfuse::Circuit(n_qubits, std::move(gs), n_params);
}

template <class T>
qfuse::BatchedState<T> make_state(const void *psi0, uint32_t n, uint32_t batch) {
    qfuse::BatchedState<T> s(n, batch);
    std::memcpy(s.components().data(), psi0, s.components().size() * sizeof(T));
    return s;
}

template <class T>
void run_gradient(const qfuse::Circuit &circuit, const void *psi0_raw, uint32_t batch,
                  const double *theta, const qfuse::PauliString &pauli, uint32_t layers,
                  uint32_t block_layers, int mode, double *loss, double *grad,
                  double *expect) {
    const auto psi0 = make_state<T>(psi0_raw, circuit.n_qubits(), batch);
    std::span<const double> th(theta, circuit.n_params());
    qfuse::GradientResult r;
    if (mode == 1) { // naive per-gate
        if (block_layers == 0) {
            r = qfuse::naive_gradient<T>(circuit, psi0, th, pauli);
        } else {
            const auto plan = qfuse::CheckpointPlan::uniform(circuit.gates().size(), layers,
                                                             block_layers);
            r = qfuse::run_checkpointed_naive<T>(circuit, psi0, th, pauli, plan);
        }
    } else {
        const auto fused = qfuse::fuse_circuit(circuit);
        const auto smode = mode == 2 ? qfuse::StorageMode::MemSave : qfuse::StorageMode::Full;
        if (block_layers == 0) {
            r = qfuse::gradient<T>(fused, psi0, th, pauli, smode);
        } else {
            const auto plan =
                qfuse::CheckpointPlan::uniform(fused.ops.size(), layers, block_layers);
            r = qfuse::run_checkpointed<T>(fused, psi0, th, pauli, plan, smode);
        }
        if (expect != nullptr) {
            const auto fw = qfuse::forward<T>(fused, psi0, th, qfuse::StorageMode::Full);
            const auto e = qfuse::expectation<T>(fw.state, pauli);
            for (uint32_t s = 0; s < batch; ++s) expect[s] = e[s];
        }
    }
    *loss = r.loss;
    for (uint32_t j = 0; j < circuit.n_params(); ++j) grad[j] = r.gradient[j];
}

} // namespace

extern "C" {

const char *ref_last_error(void) { return g_err.c_str(); }

void ref_set_threads(int threads) {
    if (threads > 0) omp_set_num_threads(threads);
}

int ref_max_threads(void) { return omp_get_max_threads(); }

void ref_set_alloc_limit(uint64_t bytes) { qfuse::set_alloc_limit(bytes); }

int ref_random_state_f64(uint32_t n, uint32_t batch, uint64_t seed, double *out) {
    return guarded([&] {
        const auto s = qfuse::new_random_state<double>(n, batch, seed);
        std::memcpy(out, s.components().data(), s.components().size() * sizeof(double));
    });
}

int ref_random_state_f32(uint32_t n, uint32_t batch, uint64_t seed, float *out) {
    return guarded([&] {
        const auto s = qfuse::new_random_state<float>(n, batch, seed);
        std::memcpy(out, s.components().data(), s.components().size() * sizeof(float));
    });
}

int ref_random_parameters(uint64_t count, uint64_t seed, double *out) {
    return guarded([&] {
        const auto t = qfuse::random_parameters(count, seed);
        std::memcpy(out, t.data(), t.size() * sizeof(double));
    });
}

// Writes up to `cap` gates; *n_gates receives the full count.
int ref_build_hea(uint32_t n, uint32_t layers, RefGate *out, uint64_t cap, uint64_t *n_gates,
                  uint32_t *n_params) {
    return guarded([&] {
        const auto c = qfuse::build_hea(n, layers);
        *n_gates = c.gates().size();
        *n_params = c.n_params();
        for (size_t i = 0; i < c.gates().size() && i < cap; ++i) {
            const auto &g = c.gates()[i];
            out[i] = RefGate{static_cast<uint8_t>(g.kind), static_cast<uint8_t>(g.axis), 0,
                             g.q0, g.q1, g.param};
        }
    });
}

int ref_parse_pauli(const char *label, uint32_t expected_n, uint64_t *x_mask, uint64_t *z_mask,
                    uint32_t *y_count) {
    return guarded([&] {
        const auto p = qfuse::parse_pauli(label, expected_n);
        *x_mask = p.x_mask;
        *z_mask = p.z_mask;
        *y_count = p.y_count;
    });
}

// precision: 0 = float (complex64), 1 = double. mode: 0 fused, 1 naive, 2 fused mem-save.
// block_layers: 0 = no checkpointing (full ledger), else run_checkpointed with
// CheckpointPlan::uniform(ops, layers, block_layers).
int ref_gradient(const RefGate *gates, uint64_t n_gates, uint32_t n_qubits, uint32_t n_params,
                 uint32_t layers, uint32_t block_layers, int precision, int mode,
                 const void *psi0, uint32_t batch, const double *theta, uint64_t x_mask,
                 uint64_t z_mask, double *loss, double *grad, double *expect) {
    return guarded([&] {
        const auto circuit = make_circuit(gates, n_gates, n_qubits, n_params);
        const qfuse::PauliString pauli(n_qubits, x_mask, z_mask);
        if (precision == 0) {
            run_gradient<float>(circuit, psi0, batch, theta, pauli, layers, block_layers, mode,
                                loss, grad, expect);
        } else {
            run_gradient<double>(circuit, psi0, batch, theta, pauli, layers, block_layers,
                                 mode, loss, grad, expect);
        }
    });
}

// Final state of the fused forward (double precision), interleaved re/im.
int ref_forward_f64(const RefGate *gates, uint64_t n_gates, uint32_t n_qubits,
                    uint32_t n_params, const double *psi0, uint32_t batch,
                    const double *theta, double *out) {
    return guarded([&] {
        const auto circuit = make_circuit(gates, n_gates, n_qubits, n_params);
        const auto fused = qfuse::fuse_circuit(circuit);
        const auto s0 = make_state<double>(psi0, n_qubits, batch);
        const auto fw = qfuse::forward<double>(fused, s0, {theta, n_params},
                                               qfuse::StorageMode::Full);
        std::memcpy(out, fw.state.components().data(),
                    fw.state.components().size() * sizeof(double));
    });
}

int ref_parameter_shift(const RefGate *gates, uint64_t n_gates, uint32_t n_qubits,
                        uint32_t n_params, const double *psi0, uint32_t batch,
                        const double *theta, uint64_t x_mask, uint64_t z_mask, double *grad) {
    return guarded([&] {
        const auto circuit = make_circuit(gates, n_gates, n_qubits, n_params);
        const auto s0 = make_state<double>(psi0, n_qubits, batch);
        const qfuse::PauliString pauli(n_qubits, x_mask, z_mask);
        const auto r = qfuse::oracle::parameter_shift_gradient(circuit, s0,
                                                               {theta, n_params}, pauli);
        for (uint32_t j = 0; j < n_params; ++j) grad[j] = r.gradient[j];
    });
}

} // extern "C"
