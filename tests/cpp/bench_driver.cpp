// Host-driver integration: the reference's bench API (bench.hpp) run by the
// reference (CPU) and by qfuse::b200::run_bench (B200) on the same BenchConfig;
// our BenchReport serialised with the reference's own report_to_json /
// report_to_csv_row and parsed back (schema round trip, bench.cpp:254-442).
// Also the CLI of the B200 driver: `bench_driver --qubits 20 --layers 1000 ...`
// prints the reference's JSON report (flags of qfuse-bench, tools/qfuse_bench_main.cpp:51-78).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "qfuse/bench.hpp"
#include "qfuse_b200.hpp"
#include "qfuse_b200_bench.hpp"

using namespace qfuse;
using namespace qfuse::bench;

static int failures = 0;
static void report(const char *name, bool ok, double v) {
    std::printf("%s %s (%.3e)\n", ok ? "PASS" : "FAIL", name, v);
    if (!ok) ++failures;
}
static double rel(double a, double b) { return std::abs(a - b) / std::max(1.0, std::abs(b)); }

static void compare(const char *name, const BenchConfig &c, double tol) {
    const BenchReport ours = b200::run_bench(c);
    const BenchReport ref = bench::run_bench(c);
    const double d = std::max(rel(ours.loss, ref.loss), rel(ours.gradient_checksum, ref.gradient_checksum));
    report(name, d <= tol && ours.config.observable == ref.config.observable, d);
    // the reference's serialisers take our report as is, and round-trip it
    const BenchReport back = report_from_json(report_to_json(ours));
    report((std::string(name) + " json round trip").c_str(), deterministic_fields_equal(back, ours), 0);
    const auto rows = reports_from_csv(reports_to_csv({ours}));
    report((std::string(name) + " csv round trip").c_str(),
           rows.size() == 1 && deterministic_fields_equal(rows[0], ours), 0);
}

static int run_tests() {
    set_alloc_limit(std::size_t{64} << 30);
    BenchConfig c; // BASELINE config 1: 4q x 4L, batch 8, IXYZ
    c.qubits = 4; c.layers = 4; c.batch = 8; c.reps = 2; c.warmup = 1;
    compare("config1 fused", c, 1e-4);
    c.mode = Mode::Naive;
    compare("config1 naive", c, 1e-4);
    c.mode = Mode::Fused;
    c.precision = Precision::Double;
    compare("config1 double", c, 1e-10);
    c.precision = Precision::Single;
    BenchConfig s = c; // 16q, block 2, MemSave vs the reference's MemSave (C10)
    s.qubits = 16; s.layers = 4; s.batch = 2; s.block = 2; s.mode = Mode::FusedMemSave;
    compare("16q memsave block 2", s, 5e-3);
    BenchConfig h = c; // build_hea_shape replica (circuit.cpp:116-143)
    h.qubits = 8; h.layers = 2; h.shape_qubits = 20;
    compare("shape replica 8q/20", h, 1e-4);
    const auto scan = b200::scan_blocks(BenchConfig{6, 8, 2}, {1, 2, 4, 8});
    bool same = scan.size() == 4;
    for (const auto &r : scan) same = same && rel(r.gradient_checksum, scan[0].gradient_checksum) <= 1e-4;
    report("scan_blocks 1,2,4,8", same, 0);
    bool threw = false;
    try { b200::scan_blocks(BenchConfig{6, 8, 2}, {3}); } catch (const std::invalid_argument &) { threw = true; }
    report("scan_blocks 3 -> invalid_argument", threw, 0);
    std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "ALL PASSED", failures);
    return failures ? 1 : 0;
}

int main(int argc, char **argv) {
    if (argc == 1 || (argc == 2 && !std::strcmp(argv[1], "--selftest"))) return run_tests();
    BenchConfig c;
    std::vector<std::uint32_t> scan;
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) throw std::invalid_argument("missing value for " + a);
            return argv[++i];
        };
        if (a == "--qubits") c.qubits = std::stoul(val());
        else if (a == "--layers") c.layers = std::stoul(val());
        else if (a == "--batch") c.batch = std::stoul(val());
        else if (a == "--shape") c.shape_qubits = std::stoul(val());
        else if (a == "--mode") c.mode = mode_from_string(val());
        else if (a == "--block") c.block = std::stoul(val());
        else if (a == "--precision") c.precision = val() == "double" ? Precision::Double : Precision::Single;
        else if (a == "--seed") c.seed = std::stoull(val());
        else if (a == "--observable") c.observable = val();
        else if (a == "--reps") c.reps = std::stoul(val());
        else if (a == "--warmup") c.warmup = std::stoul(val());
        else if (a == "--format") c.format = val();
        else if (a == "--scan-blocks") {
            const std::string v = val();
            size_t p = 0;
            while (p < v.size()) {
                const size_t q = v.find(',', p);
                scan.push_back(std::stoul(v.substr(p, q - p)));
                p = q == std::string::npos ? v.size() : q + 1;
            }
        } else if (a == "--device") b200::set_device(std::stoi(val()));
        else throw std::invalid_argument("unknown flag " + a);
    }
    try {
        if (scan.empty()) {
            const BenchReport r = b200::run_bench(c);
            std::puts(c.format == "csv" ? (csv_header() + "\n" + report_to_csv_row(r)).c_str()
                                        : report_to_json(r).c_str());
        } else {
            const auto rs = b200::scan_blocks(c, scan);
            std::puts(c.format == "csv" ? reports_to_csv(rs).c_str() : reports_to_json(rs).c_str());
        }
    } catch (const CapacityError &e) { // exit codes of qfuse_bench_main.cpp:110-116
        std::fprintf(stderr, "capacity: %s\n", e.what());
        return 3;
    } catch (const std::invalid_argument &e) {
        std::fprintf(stderr, "config: %s\n", e.what());
        return 2;
    }
    return 0;
}
