// qfuse-b200 as a link-time drop-in for the reference engine.
//
// The reference's callers (its host driver bench.cpp:95-178, its tests, user
// code) call the engine templates declared in qfuse/engine.hpp and
// qfuse/checkpoint.hpp; the reference defines them in engine.cpp /
// checkpoint.cpp as explicit instantiations for float and double
// (engine.cpp:896-944, checkpoint.cpp:190-213). This file defines the same
// specializations -- same mangled symbols -- on top of the qfuse::b200 shim,
// so the UNMODIFIED reference driver and caller objects, linked against
// libqfuse_engine_b200.so instead of engine.o + checkpoint.o, run the
// gradients on the B200. Nothing of the CPU engine is linked: the library is
// built with -Wl,--no-undefined against the reference's host IR only
// (common, statevec, circuit, fusion), see tests/cpp/Makefile.
//
//   qfuse::gradient<T>              engine.hpp:139-142
//   qfuse::naive_gradient<T>        engine.hpp:146-149
//   qfuse::forward<float>           engine.hpp:131-133 (forward<double> is not provided)
//   qfuse::run_checkpointed<T>      checkpoint.hpp:65-69
//   qfuse::run_checkpointed_naive<T> checkpoint.hpp:73-79
//
// checkpoint.cpp also holds three small host-side planning functions the
// driver needs (CheckpointPlan::uniform and the ledger-unit models
// model_native / model_fused / optimal_block, checkpoint.cpp:24-77); they are restated here
// because that object file cannot be linked without the CPU engine.
#include <cmath>
#include <stdexcept>
#include <string>

#include "qfuse_b200.hpp"

namespace qfuse {

namespace {
void check_layers(std::uint32_t layers, std::uint32_t block_layers) { // checkpoint.cpp:24-34
    if (layers == 0 || block_layers == 0)
        throw std::invalid_argument("checkpoint: layer counts must be positive");
    if (layers % block_layers != 0)
        throw std::invalid_argument("checkpoint: block size " + std::to_string(block_layers) +
                                    " does not divide layer count " + std::to_string(layers));
}
} // namespace

// checkpoint.cpp:38-49
CheckpointPlan CheckpointPlan::uniform(std::size_t total_ops, std::uint32_t layers,
                                       std::uint32_t block_layers) {
    check_layers(layers, block_layers);
    if (total_ops == 0 || total_ops % layers != 0)
        throw std::invalid_argument("checkpoint: op count is not layer-periodic");
    CheckpointPlan p;
    p.layers = layers;
    p.block_layers = block_layers;
    p.ops_per_layer = total_ops / layers;
    return p;
}

// Ledger-unit models of the host capacity check (checkpoint.cpp:50-77): per-gate
// ledger of one block plus one slot per block; fused: the ledger of one block of
// variational ops (a fused op per <= max_constituents variational gates), MemSave
// entries count half.
double model_native(std::uint32_t block_layers, std::uint32_t var_gates_per_layer,
                    std::uint32_t const_gates_per_layer, std::uint32_t layers) {
    check_layers(layers, block_layers);
    return double(var_gates_per_layer + const_gates_per_layer) * block_layers +
           double(layers) / block_layers;
}

double model_fused(std::uint32_t block_layers, std::uint32_t var_gates_per_layer,
                   std::uint32_t max_constituents, std::uint32_t layers, StorageMode mode) {
    check_layers(layers, block_layers);
    if (max_constituents == 0) throw std::invalid_argument("model_fused: constituent cap must be positive");
    const double unit = mode == StorageMode::MemSave ? 0.5 : 1.0;
    const std::uint32_t entries = (var_gates_per_layer + max_constituents - 1) / max_constituents;
    return entries * unit * block_layers + double(layers) / block_layers;
}

// checkpoint.cpp:72-77: the block size minimising slots + ledger.
double optimal_block(double units_per_layer, std::uint32_t layers) {
    if (units_per_layer <= 0.0)
        throw std::invalid_argument("optimal_block: units per layer must be positive");
    return std::sqrt(double(layers) / units_per_layer);
}

template <>
GradientResult gradient<float>(const FusedCircuit &fused, const BatchedState<float> &psi0,
                               std::span<const double> theta, const PauliString &pauli, StorageMode mode,
                               MemoryAccountant *accountant) {
    return b200::gradient(fused, psi0, theta, pauli, mode, accountant);
}
template <>
GradientResult gradient<double>(const FusedCircuit &fused, const BatchedState<double> &psi0,
                                std::span<const double> theta, const PauliString &pauli, StorageMode mode,
                                MemoryAccountant *accountant) {
    return b200::gradient(fused, psi0, theta, pauli, mode, accountant);
}

template <>
GradientResult naive_gradient<float>(const Circuit &circuit, const BatchedState<float> &psi0,
                                     std::span<const double> theta, const PauliString &pauli,
                                     MemoryAccountant *accountant) {
    return b200::naive_gradient(circuit, psi0, theta, pauli, accountant);
}
template <>
GradientResult naive_gradient<double>(const Circuit &circuit, const BatchedState<double> &psi0,
                                      std::span<const double> theta, const PauliString &pauli,
                                      MemoryAccountant *accountant) {
    return b200::naive_gradient(circuit, psi0, theta, pauli, accountant);
}

template <>
ForwardResult<float> forward<float>(const FusedCircuit &fused, const BatchedState<float> &psi0,
                                    std::span<const double> theta, StorageMode mode,
                                    MemoryAccountant *accountant) {
    return b200::forward(fused, psi0, theta, mode, accountant);
}

template <>
GradientResult run_checkpointed<float>(const FusedCircuit &fused, const BatchedState<float> &psi0,
                                       std::span<const double> theta, const PauliString &pauli,
                                       const CheckpointPlan &plan, StorageMode mode,
                                       MemoryAccountant *accountant) {
    return b200::run_checkpointed(fused, psi0, theta, pauli, plan, mode, accountant);
}
template <>
GradientResult run_checkpointed<double>(const FusedCircuit &fused, const BatchedState<double> &psi0,
                                        std::span<const double> theta, const PauliString &pauli,
                                        const CheckpointPlan &plan, StorageMode mode,
                                        MemoryAccountant *accountant) {
    return b200::run_checkpointed(fused, psi0, theta, pauli, plan, mode, accountant);
}

template <>
GradientResult run_checkpointed_naive<float>(const Circuit &circuit, const BatchedState<float> &psi0,
                                             std::span<const double> theta, const PauliString &pauli,
                                             const CheckpointPlan &plan, MemoryAccountant *accountant) {
    return b200::run_checkpointed_naive(circuit, psi0, theta, pauli, plan, accountant);
}
template <>
GradientResult run_checkpointed_naive<double>(const Circuit &circuit, const BatchedState<double> &psi0,
                                              std::span<const double> theta, const PauliString &pauli,
                                              const CheckpointPlan &plan, MemoryAccountant *accountant) {
    return b200::run_checkpointed_naive(circuit, psi0, theta, pauli, plan, accountant);
}

} // namespace qfuse
