// qfuse-b200 C++ drop-in for the reference's hot path.
//
// Same types and signatures as the reference engine (compile against the
// reference headers, proj/include), executed on a B200 through the C-ABI in
// include/qfuse_b200.h:
//
//   qfuse::b200::gradient          <- qfuse::gradient<float>         engine.hpp:139-142
//   qfuse::b200::run_checkpointed  <- qfuse::run_checkpointed<float> checkpoint.hpp:65-69
//   qfuse::b200::naive_gradient    <- qfuse::naive_gradient<float>   engine.hpp:146-149
//   qfuse::b200::run_checkpointed_naive <- run_checkpointed_naive<float> checkpoint.hpp:73-79
//   and the BatchedState<double> overloads <- the <double> instantiations
//   (engine.cpp:942, checkpoint.cpp:196-213), complex128 on the device.
//
// A caller switches by replacing `qfuse::gradient<float>(...)` with
// `qfuse::b200::gradient(...)`. Errors are rethrown as the
// reference's exception types: std::invalid_argument (C-ABI code 2),
// qfuse::CapacityError (3), std::runtime_error (4).
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "qfuse/checkpoint.hpp"
#include "qfuse/circuit.hpp"
#include "qfuse/engine.hpp"
#include "qfuse/fusion.hpp"
#include "qfuse/statevec.hpp"

namespace qfuse::b200 {

// CUDA device used by the calls of this thread (default 0, or $QFUSE_B200_DEVICE).
void set_device(int device);
// Batch-sharded multi-GPU for this thread's gradient / run_checkpointed calls
// (complex64): the samples are split over `devices` in order and [grad | loss]
// is summed with one NCCL all-reduce (qf_gradient_c64_multi). An
// empty list (default) or one device = the single-device path. The per-gate
// calls and complex128 stay on set_device's device.
void set_devices(const std::vector<int> &devices);

// forward<float> (engine.hpp:131-133): the final state before the observable,
// amplitude for amplitude the reference's (global phase included). The ledger
// of the result is empty: the device never stores per-op states.
ForwardResult<float> forward(const FusedCircuit &fused, const BatchedState<float> &psi0,
                             std::span<const double> theta, StorageMode mode,
                             MemoryAccountant *accountant = nullptr);

GradientResult gradient(const FusedCircuit &fused, const BatchedState<float> &psi0,
                        std::span<const double> theta, const PauliString &pauli,
                        StorageMode mode, MemoryAccountant *accountant = nullptr);

GradientResult run_checkpointed(const FusedCircuit &fused, const BatchedState<float> &psi0,
                                std::span<const double> theta, const PauliString &pauli,
                                const CheckpointPlan &plan, StorageMode mode,
                                MemoryAccountant *accountant = nullptr);

GradientResult naive_gradient(const Circuit &circuit, const BatchedState<float> &psi0,
                              std::span<const double> theta, const PauliString &pauli,
                              MemoryAccountant *accountant = nullptr);

GradientResult run_checkpointed_naive(const Circuit &circuit, const BatchedState<float> &psi0,
                                      std::span<const double> theta, const PauliString &pauli,
                                      const CheckpointPlan &plan,
                                      MemoryAccountant *accountant = nullptr);

// complex128 (the reference's double instantiations).
GradientResult gradient(const FusedCircuit &fused, const BatchedState<double> &psi0,
                        std::span<const double> theta, const PauliString &pauli,
                        StorageMode mode, MemoryAccountant *accountant = nullptr);

GradientResult run_checkpointed(const FusedCircuit &fused, const BatchedState<double> &psi0,
                                std::span<const double> theta, const PauliString &pauli,
                                const CheckpointPlan &plan, StorageMode mode,
                                MemoryAccountant *accountant = nullptr);

GradientResult naive_gradient(const Circuit &circuit, const BatchedState<double> &psi0,
                              std::span<const double> theta, const PauliString &pauli,
                              MemoryAccountant *accountant = nullptr);

GradientResult run_checkpointed_naive(const Circuit &circuit, const BatchedState<double> &psi0,
                                      std::span<const double> theta, const PauliString &pauli,
                                      const CheckpointPlan &plan,
                                      MemoryAccountant *accountant = nullptr);

} // namespace qfuse::b200
