// Drop-in parity: the SAME C++ calling code against the reference engine
// (CPU, qfuse::gradient<float> etc.) and against qfuse::b200 (B200, C-ABI).
// Criteria follow tests/acceptance.cpp (rel_diff :63-73); fp32 tolerance 1e-4.
#include <cmath>
#include <cstdio>
#include <span>
#include <stdexcept>
#include <vector>

#include "qfuse/checkpoint.hpp"
#include "qfuse/circuit.hpp"
#include "qfuse/engine.hpp"
#include "qfuse/fusion.hpp"
#include "qfuse/statevec.hpp"
#include "qfuse_b200.hpp"

using namespace qfuse;

static int failures = 0;

static double rel_diff(const std::vector<double> &got, const std::vector<double> &want) {
    double scale = 0, diff = 0;
    for (double w : want) scale = std::max(scale, std::abs(w));
    for (size_t i = 0; i < got.size(); ++i) diff = std::max(diff, std::abs(got[i] - want[i]));
    return scale > 0 ? diff / scale : diff;
}

static void report(const char *name, bool ok, double v) {
    std::printf("%s %s (%.3e)\n", ok ? "PASS" : "FAIL", name, v);
    if (!ok) ++failures;
}

static void compare(const char *name, const GradientResult &a, const GradientResult &b) {
    const double g = rel_diff(a.gradient, b.gradient);
    const double l = std::abs(a.loss - b.loss) / std::max(1.0, std::abs(b.loss));
    report(name, g <= 1e-4 && l <= 1e-4, std::max(g, l));
}

int main() {
    set_alloc_limit(std::size_t{64} << 30);
    {   // BASELINE config 1: 4q x 4L, batch 8, IXYZ
        Circuit c = build_hea(4, 4);
        const auto theta = random_parameters(c.n_params(), 1235);
        const auto psi0 = new_random_state<float>(4, 8, 1234);
        const auto pauli = parse_pauli(repeated_ixyz_label(4));
        const auto fused = fuse_circuit(c);
        compare("config1 gradient", b200::gradient(fused, psi0, theta, pauli, StorageMode::Full),
                gradient<float>(fused, psi0, theta, pauli, StorageMode::Full));
    }
    {   // run_checkpointed for every block size (acceptance C8)
        Circuit c = build_hea(6, 8);
        const auto theta = random_parameters(c.n_params(), 13);
        const auto psi0 = new_random_state<float>(6, 2, 14);
        const auto pauli = parse_pauli(repeated_ixyz_label(6));
        const auto fused = fuse_circuit(c);
        for (uint32_t b : {1u, 2u, 4u, 8u}) {
            const auto plan = CheckpointPlan::uniform(fused.ops.size(), 8, b);
            char name[64];
            std::snprintf(name, sizeof name, "run_checkpointed b=%u", b);
            compare(name, b200::run_checkpointed(fused, psi0, theta, pauli, plan, StorageMode::Full),
                    run_checkpointed<float>(fused, psi0, theta, pauli, plan, StorageMode::Full));
        }
    }
    {   // streaming path (n > 12) through the same call
        Circuit c = build_hea(16, 2);
        const auto theta = random_parameters(c.n_params(), 5);
        const auto psi0 = new_random_state<float>(16, 3, 6);
        const auto pauli = parse_pauli(repeated_ixyz_label(16));
        const auto fused = fuse_circuit(c);
        const auto plan = CheckpointPlan::uniform(fused.ops.size(), 2, 1);
        compare("16q run_checkpointed", b200::run_checkpointed(fused, psi0, theta, pauli, plan, StorageMode::Full),
                run_checkpointed<float>(fused, psi0, theta, pauli, plan, StorageMode::Full));
    }
    {   // StorageMode::MemSave against the reference's MemSave and its Full fp32
        // gradient: acceptance C10 bound 5e-3 (acceptance.cpp:466-499)
        Circuit c = build_hea(16, 4);
        const auto theta = random_parameters(c.n_params(), 31);
        const auto psi0 = new_random_state<float>(16, 2, 32);
        const auto pauli = parse_pauli(repeated_ixyz_label(16));
        const auto fused = fuse_circuit(c);
        const auto plan = CheckpointPlan::uniform(fused.ops.size(), 4, 1);
        const auto ours = b200::run_checkpointed(fused, psi0, theta, pauli, plan, StorageMode::MemSave);
        const auto full = run_checkpointed<float>(fused, psi0, theta, pauli, plan, StorageMode::Full);
        const double g = rel_diff(ours.gradient, full.gradient);
        report("16q MemSave vs reference Full (C10 5e-3)", g <= 5e-3, g);
    }
    {   // complex128: the reference's gradient<double> / run_checkpointed<double> at the
        // double-precision bounds of acceptance C1/C8 (1e-10)
        Circuit c = build_hea(6, 5);
        const auto theta = random_parameters(c.n_params(), 41);
        const auto psi0 = new_random_state<double>(6, 3, 42);
        const auto pauli = parse_pauli(repeated_ixyz_label(6));
        const auto fused = fuse_circuit(c);
        const auto a = b200::gradient(fused, psi0, theta, pauli, StorageMode::Full);
        const auto b = gradient<double>(fused, psi0, theta, pauli, StorageMode::Full);
        const double g = std::max(rel_diff(a.gradient, b.gradient),
                                  std::abs(a.loss - b.loss) / std::max(1.0, std::abs(b.loss)));
        report("complex128 gradient<double> (1e-10)", g <= 1e-10, g);
        const auto plan = CheckpointPlan::uniform(fused.ops.size(), 5, 1);
        const auto cp = b200::run_checkpointed(fused, psi0, theta, pauli, plan, StorageMode::Full);
        const double h = rel_diff(cp.gradient, b.gradient);
        report("complex128 run_checkpointed<double> (1e-10)", h <= 1e-10, h);
    }
    {   // per-gate comparator: naive_gradient
        Circuit c = build_hea(5, 3);
        const auto theta = random_parameters(c.n_params(), 21);
        const auto psi0 = new_random_state<float>(5, 4, 22);
        const auto pauli = parse_pauli("ZZZZZ");
        compare("naive_gradient", b200::naive_gradient(c, psi0, theta, pauli),
                naive_gradient<float>(c, psi0, theta, pauli));
    }
    {   // error taxonomy
        Circuit c = build_hea(4, 2);
        const auto fused = fuse_circuit(c);
        const auto psi0 = new_random_state<float>(4, 2, 1);
        const auto pauli = parse_pauli("IXYZ");
        std::vector<double> short_theta(3, 0.1);
        bool ok = false;
        try { b200::gradient(fused, psi0, short_theta, pauli, StorageMode::Full); }
        catch (const std::invalid_argument &) { ok = true; }
        report("theta length -> invalid_argument", ok, 0);
        ok = false;
        const auto theta = random_parameters(c.n_params(), 2);
        try {
            const auto plan = CheckpointPlan::uniform(fused.ops.size(), 2, 2);
            CheckpointPlan bad = plan;
            bad.layers = 3;
            b200::run_checkpointed(fused, psi0, theta, pauli, bad, StorageMode::Full);
        } catch (const std::invalid_argument &) { ok = true; }
        report("plan mismatch -> invalid_argument", ok, 0);
    }
    std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "ALL PASSED", failures);
    return failures ? 1 : 0;
}
