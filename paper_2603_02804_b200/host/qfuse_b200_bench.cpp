// B200 host driver mirroring the reference's run_bench (bench.cpp:95-178).
#include "qfuse_b200_bench.hpp"

#include <chrono>
#include <cmath>
#include <stdexcept>
#include <string>

#include "qfuse_b200.hpp"

namespace qfuse::b200 {
namespace {

using bench::BenchConfig;
using bench::BenchReport;
using bench::Mode;

std::string observable_of(const BenchConfig &c) { // bench.cpp:60-63
    return c.observable.empty() ? repeated_ixyz_label(c.qubits) : c.observable;
}

// BenchConfig::validate (bench.cpp:188-220) minus the host working-set model:
// the device plan checks its own HBM budget (CapacityError, C-ABI code 3).
void validate(const BenchConfig &c) {
    if (c.qubits < 2) throw std::invalid_argument("config: need at least 2 qubits");
    if (c.layers == 0) throw std::invalid_argument("config: need at least 1 layer");
    if (c.batch == 0) throw std::invalid_argument("config: batch must be >= 1");
    if (c.shape_qubits != 0 && (c.shape_qubits < 2 || c.qubits < 3))
        throw std::invalid_argument("config: shape replica needs shape >= 2 and at least 3 qubits");
    if (c.reps == 0) throw std::invalid_argument("config: repetitions must be >= 1");
    if (c.block != 0 && c.layers % c.block != 0)
        throw std::invalid_argument("config: block " + std::to_string(c.block) +
                                    " does not divide layer count " + std::to_string(c.layers));
    if (c.format != "csv" && c.format != "json")
        throw std::invalid_argument("config: format must be csv or json");
    parse_pauli(observable_of(c), c.qubits);
}

template <class T> BenchReport run_impl(const BenchConfig &config) {
    Circuit circuit = config.shape_qubits > 0
                          ? build_hea_shape(config.qubits, config.layers, config.shape_qubits)
                          : build_hea(config.qubits, config.layers);
    circuit.theta() = random_parameters(circuit.n_params(), config.seed + 1);
    const PauliString pauli = parse_pauli(observable_of(config), config.qubits);
    const BatchedState<T> psi0 = new_random_state<T>(config.qubits, config.batch, config.seed);
    const FusedCircuit fused = fuse_circuit(circuit);
    const StorageMode mode =
        config.mode == Mode::FusedMemSave ? StorageMode::MemSave : StorageMode::Full;
    const std::size_t amp_bytes = sizeof(T) * 2;
    MemoryAccountant accountant((std::size_t{1} << config.qubits) * config.batch * amp_bytes);

    auto run_once = [&]() -> GradientResult {
        accountant.reset();
        if (config.block == 0) {
            if (config.mode == Mode::Naive)
                return naive_gradient(circuit, psi0, circuit.theta(), pauli, &accountant);
            return gradient(fused, psi0, circuit.theta(), pauli, mode, &accountant);
        }
        if (config.mode == Mode::Naive) {
            const auto plan = CheckpointPlan::uniform(circuit.gates().size(), config.layers, config.block);
            return run_checkpointed_naive(circuit, psi0, circuit.theta(), pauli, plan, &accountant);
        }
        const auto plan = CheckpointPlan::uniform(fused.ops.size(), config.layers, config.block);
        return run_checkpointed(fused, psi0, circuit.theta(), pauli, plan, mode, &accountant);
    };

    for (std::uint32_t i = 0; i < config.warmup; ++i) run_once();
    std::vector<double> wall(config.reps, 0.0);
    GradientResult last;
    for (std::uint32_t i = 0; i < config.reps; ++i) { // bench.cpp:139-146: host wall clock
        const auto t0 = std::chrono::steady_clock::now();
        last = run_once();
        const auto t1 = std::chrono::steady_clock::now();
        wall[i] = std::chrono::duration<double>(t1 - t0).count();
    }
    double mean = 0.0;
    for (const double w : wall) mean += w;
    mean /= double(config.reps);
    double var = 0.0;
    for (const double w : wall) var += (w - mean) * (w - mean);

    BenchReport report;
    report.config = config;
    report.config.observable = observable_of(config);
    report.wall_mean_s = mean;
    report.wall_stddev_s = config.reps > 1 ? std::sqrt(var / double(config.reps - 1)) : 0.0;
    report.throughput_sps = mean > 0.0 ? double(config.batch) / mean : 0.0;
    report.forward_traversals = last.stats.forward_traversals;
    report.backward_traversals = last.stats.backward_traversals;
    report.observable_traversals = last.stats.observable_traversals;
    report.ledger_peak_units = accountant.peak_units();
    report.ledger_peak_bytes = accountant.peak_bytes();
    report.loss = last.loss;
    double checksum = 0.0;
    for (const double g : last.gradient) checksum += g;
    report.gradient_checksum = checksum;
    return report;
}

} // namespace

bench::BenchReport run_bench(const bench::BenchConfig &config) {
    validate(config);
    return config.precision == Precision::Single ? run_impl<float>(config) : run_impl<double>(config);
}

std::vector<bench::BenchReport> scan_blocks(const bench::BenchConfig &config,
                                            const std::vector<std::uint32_t> &blocks) {
    if (blocks.empty()) throw std::invalid_argument("scan_blocks: empty block list");
    for (const std::uint32_t b : blocks)
        if (b == 0 || config.layers % b != 0)
            throw std::invalid_argument("scan_blocks: block " + std::to_string(b) +
                                        " does not divide layer count " + std::to_string(config.layers));
    std::vector<bench::BenchReport> out;
    for (const std::uint32_t b : blocks) {
        bench::BenchConfig c = config;
        c.block = b;
        out.push_back(b200::run_bench(c));
    }
    return out;
}

} // namespace qfuse::b200
