// Host driver CLI: the reference's own bench API (qfuse::bench::run_bench /
// scan_blocks and the report serialisers, bench.cpp, compiled from the
// reference's unmodified source) behind the flags of qfuse-bench
// (tools/qfuse_bench_main.cpp:51-78; its CLI11 front end is not vendored in
// the reference, so this file parses the same flags by hand, with the same
// exit codes, qfuse_bench_main.cpp:110-116).
//
// Built twice from this file (tests/cpp/Makefile):
//   build/tests/bench_driver_ref  linked with the reference engine (oracle/_ref): CPU
//   build/tests/bench_driver      linked with libqfuse_engine_b200.so (QF_B200): the
//                                 same driver code, every gradient on the B200
// B200-only flags: --device D, --gpus N (batch-sharded over devices 0..N-1 with
// one NCCL all-reduce, qf_gradient_c64_multi). Golden-state exchange in the
// reference's QSV1 format (dump_state / load_state, statevec.cpp:122-186):
//   --golden-out F    write forward<float>(workload) final states to F
//   --golden-check F  load F and compare it with this build's forward<float>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "qfuse/bench.hpp"
#include "qfuse/circuit.hpp"
#include "qfuse/engine.hpp"
#include "qfuse/fusion.hpp"
#include "qfuse/statevec.hpp"
#ifdef QF_B200
#include "qfuse_b200.hpp"
#endif

using namespace qfuse;
using namespace qfuse::bench;

namespace {

int failures = 0;
void report(const std::string &name, bool ok, double v) {
    std::printf("%s %s (%.3e)\n", ok ? "PASS" : "FAIL", name.c_str(), v);
    if (!ok) ++failures;
}

// Self-test of the driver integration: this build's report goes through the
// reference's JSON/CSV serialisers and back; scan_blocks validates blocks.
int run_selftest() {
    set_alloc_limit(std::size_t{64} << 30);
    BenchConfig c; // BASELINE config 1: 4q x 4L, batch 8, IXYZ
    c.qubits = 4; c.layers = 4; c.batch = 8; c.reps = 2; c.warmup = 1;
    for (const Mode m : {Mode::Fused, Mode::Naive, Mode::FusedMemSave}) {
        c.mode = m;
        const BenchReport r = run_bench(c);
        const std::string name = std::string("config1 ") + to_string(m);
        report(name + " finite", std::isfinite(r.loss) && std::isfinite(r.gradient_checksum), r.loss);
        const BenchReport back = report_from_json(report_to_json(r));
        report(name + " json round trip", deterministic_fields_equal(back, r), 0);
        const auto rows = reports_from_csv(reports_to_csv({r}));
        report(name + " csv round trip", rows.size() == 1 && deterministic_fields_equal(rows[0], r), 0);
    }
    const auto scan = scan_blocks(BenchConfig{6, 8, 2}, {1, 2, 4, 8});
    bool same = scan.size() == 4;
    for (const auto &r : scan)
        same = same && std::abs(r.gradient_checksum - scan[0].gradient_checksum) <=
                           1e-4 * std::max(1.0, std::abs(scan[0].gradient_checksum));
    report("scan_blocks 1,2,4,8", same, 0);
    bool threw = false;
    try {
        scan_blocks(BenchConfig{6, 8, 2}, {3});
    } catch (const std::invalid_argument &) {
        threw = true;
    }
    report("scan_blocks 3 -> invalid_argument", threw, 0);
    std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "ALL PASSED", failures);
    return failures ? 1 : 0;
}

// forward<float> of the run_bench workload (bench.cpp:100-108 generators).
BatchedState<float> forward_state(const BenchConfig &c) {
    Circuit circuit = c.shape_qubits > 0 ? build_hea_shape(c.qubits, c.layers, c.shape_qubits)
                                         : build_hea(c.qubits, c.layers);
    circuit.theta() = random_parameters(circuit.n_params(), c.seed + 1);
    const BatchedState<float> psi0 = new_random_state<float>(c.qubits, c.batch, c.seed);
    const FusedCircuit fused = fuse_circuit(circuit);
    return forward<float>(fused, psi0, circuit.theta(), StorageMode::Full).state;
}

} // namespace

int main(int argc, char **argv) {
    if (argc == 2 && !std::strcmp(argv[1], "--selftest")) return run_selftest();
    BenchConfig c;
    std::vector<std::uint32_t> scan;
    std::string golden_out, golden_check, emit_circuit;
    double golden_tol = 1e-5;
    try {
        for (int i = 1; i < argc; ++i) {
            const std::string a = argv[i];
            auto val = [&]() -> std::string {
                if (i + 1 >= argc) throw std::invalid_argument("missing value for " + a);
                return argv[++i];
            };
            if (a == "--qubits") c.qubits = std::stoul(val());
            else if (a == "--layers") c.layers = std::stoul(val());
            else if (a == "--batch") c.batch = std::stoul(val());
            else if (a == "--shape-qubits" || a == "--shape") c.shape_qubits = std::stoul(val());
            else if (a == "--mode") c.mode = mode_from_string(val());
            else if (a == "--block") c.block = std::stoul(val());
            else if (a == "--precision") c.precision = precision_from_string(val());
            else if (a == "--seed") c.seed = std::stoull(val());
            else if (a == "--observable") c.observable = val();
            else if (a == "--reps") c.reps = std::stoul(val());
            else if (a == "--warmup") c.warmup = std::stoul(val());
            else if (a == "--threads") c.threads = std::stoul(val());
            else if (a == "--format") c.format = val();
            else if (a == "--out") c.out = val();
            else if (a == "--scan-blocks") {
                const std::string v = val();
                size_t p = 0;
                while (p < v.size()) {
                    const size_t q = v.find(',', p);
                    scan.push_back(std::stoul(v.substr(p, q - p)));
                    p = q == std::string::npos ? v.size() : q + 1;
                }
            } else if (a == "--emit-circuit") emit_circuit = val();
            else if (a == "--golden-out") golden_out = val();
            else if (a == "--golden-check") golden_check = val();
            else if (a == "--golden-tol") golden_tol = std::stod(val());
#ifdef QF_B200
            else if (a == "--device") b200::set_device(std::stoi(val()));
            else if (a == "--gpus") {
                const int n = std::stoi(val());
                if (n < 1) throw std::invalid_argument("--gpus must be >= 1");
                std::vector<int> devs(n);
                for (int d = 0; d < n; ++d) devs[d] = d;
                b200::set_devices(devs);
            }
#endif
            else throw std::invalid_argument("unknown flag " + a);
        }
        if (!emit_circuit.empty()) { // qfuse_bench_main.cpp:91-97
            std::ofstream os(emit_circuit);
            if (!os) throw std::invalid_argument("cannot open circuit file: " + emit_circuit);
            write_circuit(os, build_hea(c.qubits, c.layers));
        }
        if (!golden_out.empty() || !golden_check.empty()) {
            const BatchedState<float> mine = forward_state(c);
            if (!golden_out.empty()) {
                std::ofstream os(golden_out, std::ios::binary);
                if (!os) throw std::invalid_argument("cannot open " + golden_out);
                dump_state(mine, os);
                std::printf("wrote %s: %u samples x 2^%u amplitudes\n", golden_out.c_str(), mine.batch(),
                            mine.n_qubits());
            }
            if (!golden_check.empty()) {
                std::ifstream is(golden_check, std::ios::binary);
                if (!is) throw std::invalid_argument("cannot open " + golden_check);
                const BatchedState<float> gold = load_state<float>(is);
                if (gold.n_qubits() != mine.n_qubits() || gold.batch() != mine.batch())
                    throw std::invalid_argument("golden state shape mismatch");
                double d = 0.0;
                const auto a = gold.components(), b = mine.components();
                for (size_t k = 0; k < a.size(); ++k) d = std::max(d, double(std::abs(a[k] - b[k])));
                std::printf("golden max |diff| %.3e (tol %.1e)\n", d, golden_tol);
                if (!(d <= golden_tol)) return 1;
            }
            return 0;
        }
        std::string text;
        if (scan.empty()) {
            const BenchReport r = run_bench(c);
            text = c.format == "json" ? report_to_json(r) : reports_to_csv({r});
        } else {
            const auto rs = scan_blocks(c, scan);
            text = c.format == "json" ? reports_to_json(rs) : reports_to_csv(rs);
        }
        if (c.out.empty()) {
            std::puts(text.c_str());
        } else {
            std::ofstream os(c.out);
            if (!os) throw std::invalid_argument("cannot open output file: " + c.out);
            os << text << '\n';
        }
    } catch (const CapacityError &e) { // exit codes of qfuse_bench_main.cpp:110-116
        std::fprintf(stderr, "capacity error: %s\n", e.what());
        return 3;
    } catch (const std::exception &e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
    return 0;
}
