// qfuse-b200 C++ drop-in (see qfuse_b200.hpp). Converts the reference's host
// types to the C-ABI: flatten(fused) (fusion.cpp:103-125) -> qf_gate[],
// BatchedState components (statevec.hpp:74-76) -> float*, PauliString masks,
// CheckpointPlan -> (layers, block_layers), and RunStats <- qf_stats.
#include "qfuse_b200.hpp"

#include <algorithm>
#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/qfuse_b200.h"

namespace qfuse::b200 {
namespace {

thread_local int t_device = -1;
thread_local std::vector<int> t_devices; // > 1 entries: batch-sharded multi-GPU

struct CtxDeleter {
    void operator()(qf_ctx *c) const { qf_ctx_destroy(c); }
};

qf_ctx *context() {
    thread_local std::unique_ptr<qf_ctx, CtxDeleter> ctx;
    thread_local int ctx_device = -1;
    int dev = t_device;
    if (dev < 0) {
        const char *e = std::getenv("QFUSE_B200_DEVICE");
        dev = e ? std::atoi(e) : 0;
    }
    if (!ctx || ctx_device != dev) {
        qf_ctx *c = nullptr;
        const int rc = qf_ctx_create(dev, &c);
        if (rc != QF_OK) throw std::runtime_error(std::string("qfuse-b200: ") + qf_last_error());
        ctx.reset(c);
        ctx_device = dev;
    }
    return ctx.get();
}

void check(int rc) {
    if (rc == QF_OK) return;
    const std::string msg = qf_last_error();
    if (rc == QF_EINVAL) throw std::invalid_argument(msg);
    if (rc == QF_ECAPACITY) throw CapacityError(msg);
    throw std::runtime_error(msg);
}

std::vector<qf_gate> to_gates(const std::vector<Gate> &gates) {
    std::vector<qf_gate> out;
    out.reserve(gates.size());
    for (const Gate &g : gates) {
        qf_gate q{};
        q.kind = static_cast<uint8_t>(g.kind);
        q.axis = static_cast<uint8_t>(g.axis);
        q.q0 = g.q0;
        q.q1 = g.q1;
        q.param = g.param;
        out.push_back(q);
    }
    return out;
}

GradientResult call(bool pergate, const std::vector<Gate> &flat, uint32_t n_qubits,
                    uint32_t n_params, uint32_t layers, uint32_t block_layers,
                    const BatchedState<float> &psi0, std::span<const double> theta,
                    const PauliString &pauli, MemoryAccountant *accountant,
                    StorageMode mode = StorageMode::Full) {
    if (psi0.n_qubits() != pauli.n_qubits)
        throw std::invalid_argument("engine: state qubit count mismatch"); // engine.cpp:438-442
    if (theta.size() != n_params)
        throw std::invalid_argument("gradient: theta length mismatch"); // engine.cpp:721-723
    const auto gates = to_gates(flat);
    GradientResult r;
    r.gradient.assign(n_params, 0.0);
    qf_stats st{};
    if (pergate) {
        check(qf_gradient_pergate_c64(context(), gates.data(), gates.size(), n_qubits, n_params, layers,
                                      block_layers, psi0.components().data(), psi0.batch(), theta.data(),
                                      pauli.x_mask, pauli.z_mask, &r.loss, r.gradient.data(), nullptr, &st));
    } else {
        const uint32_t storage = mode == StorageMode::MemSave ? QF_STORAGE_MEMSAVE : QF_STORAGE_FULL;
        if (t_devices.size() > 1)
            check(qf_gradient_c64_multi(int(t_devices.size()), t_devices.data(), gates.data(), gates.size(),
                                        n_qubits, n_params, layers, block_layers, storage,
                                        psi0.components().data(), psi0.batch(), theta.data(), pauli.x_mask,
                                        pauli.z_mask, &r.loss, r.gradient.data(), nullptr, &st));
        else
            check(qf_gradient_c64_ex(context(), gates.data(), gates.size(), n_qubits, n_params, layers,
                                     block_layers, storage, psi0.components().data(), psi0.batch(),
                                     theta.data(), pauli.x_mask, pauli.z_mask, &r.loss, r.gradient.data(),
                                     nullptr, &st));
    }
    r.stats.forward_traversals = st.forward_passes;
    r.stats.backward_traversals = st.backward_passes;
    r.stats.observable_traversals = st.observable_passes;
    // stored state vectors: checkpoint slots (+1 working store), in state units
    // (MemSave slots count half, accounting.hpp:25-61 / engine.hpp:47)
    const double slots = st.stages ? double(st.stages / std::max(1u, st.ckpt_layers)) : 0.0;
    r.stats.ledger_peak_units =
        st.resident ? 0.0 : (mode == StorageMode::MemSave ? 0.5 * std::max(0.0, slots - 1) + 1.0 : slots + 1.0);
    if (accountant != nullptr) {
        accountant->add(r.stats.ledger_peak_units);
        accountant->release(r.stats.ledger_peak_units);
    }
    return r;
}

// complex128: gradient/run_checkpointed run the fused fp64 segments
// (qf_gradient_c128), naive_gradient/run_checkpointed_naive the fp64 per-gate
// path (qf_gradient_pergate_c128). MemSave has no effect there (no slots are
// stored), as in the reference at double where the narrowed type is float
// (statevec.hpp narrow_traits<double>).
GradientResult call_c128(bool naive, const std::vector<Gate> &flat, uint32_t n_qubits,
                         uint32_t n_params, uint32_t layers, uint32_t block_layers,
                         const BatchedState<double> &psi0, std::span<const double> theta,
                         const PauliString &pauli, MemoryAccountant *accountant) {
    if (psi0.n_qubits() != pauli.n_qubits)
        throw std::invalid_argument("engine: state qubit count mismatch"); // engine.cpp:438-442
    if (theta.size() != n_params)
        throw std::invalid_argument("gradient: theta length mismatch"); // engine.cpp:721-723
    const auto gates = to_gates(flat);
    GradientResult r;
    r.gradient.assign(n_params, 0.0);
    qf_stats st{};
    check((naive ? qf_gradient_pergate_c128 : qf_gradient_c128)(
        context(), gates.data(), gates.size(), n_qubits, n_params, layers, block_layers,
        psi0.components().data(), psi0.batch(), theta.data(), pauli.x_mask, pauli.z_mask, &r.loss,
        r.gradient.data(), nullptr, &st));
    r.stats.forward_traversals = st.forward_passes;
    r.stats.backward_traversals = st.backward_passes;
    r.stats.observable_traversals = st.observable_passes;
    r.stats.ledger_peak_units = 1.0; // the working store only
    if (accountant != nullptr) {
        accountant->add(r.stats.ledger_peak_units);
        accountant->release(r.stats.ledger_peak_units);
    }
    return r;
}

} // namespace

void set_device(int device) { t_device = device; }

void set_devices(const std::vector<int> &devices) {
    t_devices = devices;
    if (devices.size() == 1) t_device = devices[0];
}

ForwardResult<float> forward(const FusedCircuit &fused, const BatchedState<float> &psi0,
                             std::span<const double> theta, StorageMode, MemoryAccountant *accountant) {
    if (theta.size() != fused.n_params)
        throw std::invalid_argument("forward: theta length mismatch");
    const auto gates = to_gates(flatten(fused));
    ForwardResult<float> r{BatchedState<float>(psi0.n_qubits(), psi0.batch()), {}, {}};
    qf_stats st{};
    check(qf_forward_c64(context(), gates.data(), gates.size(), fused.n_qubits, fused.n_params, 0,
                         psi0.components().data(), psi0.batch(), theta.data(),
                         r.state.components().data(), &st));
    r.stats.forward_traversals = st.forward_passes;
    if (accountant != nullptr) { // the working store only
        accountant->add(1.0);
        accountant->release(1.0);
    }
    return r;
}

GradientResult gradient(const FusedCircuit &fused, const BatchedState<double> &psi0,
                        std::span<const double> theta, const PauliString &pauli,
                        StorageMode, MemoryAccountant *accountant) {
    return call_c128(false, flatten(fused), fused.n_qubits, fused.n_params, 0, 0, psi0, theta, pauli, accountant);
}

GradientResult run_checkpointed(const FusedCircuit &fused, const BatchedState<double> &psi0,
                                std::span<const double> theta, const PauliString &pauli,
                                const CheckpointPlan &plan, StorageMode, MemoryAccountant *accountant) {
    if (plan.ops_per_layer * plan.layers != fused.ops.size()) // checkpoint.cpp:149-151
        throw std::invalid_argument("run_checkpointed: plan does not cover the circuit");
    return call_c128(false, flatten(fused), fused.n_qubits, fused.n_params, plan.layers, plan.block_layers,
                     psi0, theta, pauli, accountant);
}

GradientResult naive_gradient(const Circuit &circuit, const BatchedState<double> &psi0,
                              std::span<const double> theta, const PauliString &pauli,
                              MemoryAccountant *accountant) {
    return call_c128(true, circuit.gates(), circuit.n_qubits(), circuit.n_params(), 0, 0, psi0, theta,
                     pauli, accountant);
}

GradientResult gradient(const FusedCircuit &fused, const BatchedState<float> &psi0,
                        std::span<const double> theta, const PauliString &pauli,
                        StorageMode mode, MemoryAccountant *accountant) {
    const auto flat = flatten(fused);
    return call(false, flat, fused.n_qubits, fused.n_params, 0, 0, psi0, theta, pauli,
                accountant, mode);
}

GradientResult run_checkpointed(const FusedCircuit &fused, const BatchedState<float> &psi0,
                                std::span<const double> theta, const PauliString &pauli,
                                const CheckpointPlan &plan, StorageMode mode,
                                MemoryAccountant *accountant) {
    if (plan.ops_per_layer * plan.layers != fused.ops.size()) // checkpoint.cpp:149-151
        throw std::invalid_argument("run_checkpointed: plan does not cover the circuit");
    const auto flat = flatten(fused);
    return call(false, flat, fused.n_qubits, fused.n_params, plan.layers, plan.block_layers, psi0,
                theta, pauli, accountant, mode);
}

GradientResult run_checkpointed_naive(const Circuit &circuit, const BatchedState<float> &psi0,
                                      std::span<const double> theta, const PauliString &pauli,
                                      const CheckpointPlan &plan, MemoryAccountant *accountant) {
    if (plan.ops_per_layer * plan.layers != circuit.gates().size()) // checkpoint.cpp:172-175
        throw std::invalid_argument("run_checkpointed_naive: plan does not cover the circuit");
    return call(true, circuit.gates(), circuit.n_qubits(), circuit.n_params(), plan.layers,
                plan.block_layers, psi0, theta, pauli, accountant);
}

GradientResult run_checkpointed_naive(const Circuit &circuit, const BatchedState<double> &psi0,
                                      std::span<const double> theta, const PauliString &pauli,
                                      const CheckpointPlan &plan, MemoryAccountant *accountant) {
    if (plan.ops_per_layer * plan.layers != circuit.gates().size())
        throw std::invalid_argument("run_checkpointed_naive: plan does not cover the circuit");
    return call_c128(true, circuit.gates(), circuit.n_qubits(), circuit.n_params(), plan.layers,
                     plan.block_layers, psi0, theta, pauli, accountant);
}

GradientResult naive_gradient(const Circuit &circuit, const BatchedState<float> &psi0,
                              std::span<const double> theta, const PauliString &pauli,
                              MemoryAccountant *accountant) {
    return call(true, circuit.gates(), circuit.n_qubits(), circuit.n_params(), 0, 0, psi0, theta,
                pauli, accountant);
}

} // namespace qfuse::b200
