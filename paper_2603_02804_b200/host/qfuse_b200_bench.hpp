// qfuse-b200 host driver: the reference's bench entry points on the B200.
//
//   qfuse::b200::run_bench   <- qfuse::bench::run_bench   bench.hpp:79, bench.cpp:95-178
//   qfuse::b200::scan_blocks <- qfuse::bench::scan_blocks bench.hpp:83-84, bench.cpp:228-250
//
// Same BenchConfig in, same BenchReport out (bench.hpp:29-68): the workload is
// built with the reference's own generators (build_hea / build_hea_shape,
// random_parameters(M, seed + 1), new_random_state<T>(n, B, seed), the IXYZ
// observable), `warmup` untimed and `reps` timed runs through qfuse::b200, the
// counters of the last run. The reference's report serialisers
// (report_to_json / report_to_csv_row, bench.cpp:254-442) take the result as is.
// Differences: traversal counters are the device's fused passes (qf_stats),
// ledger_peak_units counts checkpoint slots (MemSave slots as half units), and
// the capacity check is the device's HBM budget, not the host alloc limit.
#pragma once

#include <vector>

#include "qfuse/bench.hpp"

namespace qfuse::b200 {

bench::BenchReport run_bench(const bench::BenchConfig &config);
std::vector<bench::BenchReport> scan_blocks(const bench::BenchConfig &config,
                                            const std::vector<std::uint32_t> &blocks);

} // namespace qfuse::b200
