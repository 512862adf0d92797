// Host planner: flattened gate list -> device stages, sections and passes.
// Theta-independent; a plan is reused across gradient calls.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/qfuse_b200.h"
#include "qf_internal.h"

namespace qfb {

// Error taxonomy of the reference (common.hpp:32-35, engine.cpp:438-442):
// invalid_argument -> QF_EINVAL, CapacityError -> QF_ECAPACITY.
struct CapacityError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct PassLayout {
    int row_start;     // first qubit of the 8 row bits
    int tile_lo_bits;  // bits between column and rows
    int tile_hi_bits;  // bits above the rows
    uint32_t rot_mask; // local bits rotated in this pass
    int qmap[12];      // local bit -> qubit
    bool has_diag;     // pass A
};

struct Plan {
    uint32_t n = 0, n_params = 0, layers = 0, batch = 0;
    uint64_t x_mask = 0, z_mask = 0;
    uint32_t y_count = 0;
    // stages and diagonals
    uint32_t stages = 0;
    std::vector<CzSet> czsets;     // distinct CZ sets (index 0.. )
    std::vector<int> stage_cz;     // [stages] -> czsets index or -1
    int final_cz = -1;             // index or -1
    // sections (one per single-qubit run)
    std::vector<uint32_t> sec_q, sec_stage, sec_alpha_row, sec_off, sec_gates;
    // schedule
    bool resident = false;         // n <= 12: one kernel per gradient
    std::vector<PassLayout> passes;// streaming: A, B, (C)
    uint32_t ckpt_stages = 1;      // k in stages
    uint32_t ckpt_layers = 0;      // k in layers as reported
    uint32_t n_slots = 0;
    // per-gate comparator: flattened gates kept as given
    std::vector<qf_gate> gates;
};

// Builds a plan (throws std::invalid_argument / CapacityError with the
// reference's messages).
Plan make_plan(const qf_gate *gates, size_t n_gates, uint32_t n_qubits, uint32_t n_params,
               uint32_t layers, uint32_t ckpt_layers, uint32_t batch, uint64_t x_mask,
               uint64_t z_mask);

CzSet make_czset(const std::vector<std::pair<uint32_t, uint32_t>> &pairs);

} // namespace qfb
