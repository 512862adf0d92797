// Host planner: flattened gate list -> device stages, sections and passes.
// Theta-independent; a plan is reused across gradient calls.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/qfuse_b200.h"
#include "qf_internal.h"

namespace qfb {

// Error taxonomy of the reference (common.hpp:32-35, engine.cpp:438-442):
// invalid_argument -> QF_EINVAL, CapacityError -> QF_ECAPACITY.
struct CapacityError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// Which 12 qubits a tile keeps resident, and how the rest index tiles.
struct PassLayout {
    int row_start = 4;    // first qubit of the 8 row bits
    int tile_lo_bits = 0; // tile bits between column and rows (qubits 4..row_start-1)
    int tile_hi_bits = 0; // tile bits above the rows (qubits row_start+8..n-1)
    uint32_t rot_mask = 0;// local bits rotated in this layout
    int qmap[12] = {};    // local bit -> qubit (-1: sample bit, resident layout only)
    int gd = 0;           // group phase that applies the diagonal
    int dq[28] = {};      // diag-group view: qubit of reg 0..3, thr 0..7, tile 0..15
    std::vector<int> tile_qubits;
};

// One forward pass: Ry_{s0}(X) -> D_{sd} -> Ry_{s1}(X) on layout X.
struct PassStep {
    int layout = 0;
    int s0 = -1, s1 = -1, sd = -1;
    int nph = 0;
    PassPhase ph[6] = {};
    uint32_t rot0 = 0, rot1 = 0; // local bits rotated in round 0 / 1 (0, 0: the layout's rot_mask)
};

struct Plan {
    uint32_t n = 0, n_params = 0, layers = 0, batch = 0;
    uint64_t x_mask = 0, z_mask = 0;
    uint32_t y_count = 0;
    // stages
    uint32_t stages = 0;
    std::vector<std::vector<std::pair<uint32_t, uint32_t>>> czsets; // distinct CZ sets
    std::vector<int> stage_cz;     // [stages] -> czsets index or -1
    int final_cz = -1;
    // sections (one per single-qubit run)
    std::vector<uint32_t> sec_q, sec_stage, sec_alpha_row, sec_off, sec_gates;
    // schedule
    bool resident = false;         // n <= 12: one kernel per gradient
    std::vector<PassLayout> layouts; // resident: [0]; streaming: A, B, (C)
    std::vector<PassStep> steps;   // streaming forward passes
    std::vector<int> stage_layout; // layout whose pass applies D_s
    std::vector<CzTab> cztab;      // [czset][layout]
    std::vector<std::vector<uint32_t>> tileinfo; // [czset][layout]
    std::vector<CzAdj> final_adj;  // 0 or 1 entries
    // wide-group view of layout 0 (forward passes with all 12 local qubits rotated,
    // qf_pass_wide.cu): dqw[0..5] register bits, [6..11] thread bits, [12..] tile bits
    bool wide = false;
    int dqw[28] = {};
    std::vector<CzTabW> cztabw;                   // [czset]
    std::vector<std::vector<uint32_t>> tileinfow; // [czset]
    // Balanced backward (n = 20): the column group's Ry of stage s is
    // undone by the backward pass that undoes D_s, so both layouts' backward passes
    // rotate 8 + 12 qubits (kProgAlt, 4 phases each) instead of 24 / 16. The forward
    // keeps `steps`; both schedules pass through the same state after every layout-A
    // pass, where the checkpoint slots sit (slot_off = 1).
    bool alt = false;
    std::vector<PassStep> bsteps;               // backward passes (alt), same indices as steps
    std::vector<CzTab> cztab_alt;               // [czset] layout A, diagonal in group 2
    std::vector<std::vector<uint32_t>> tileinfo_alt; // [czset]
    int dq_alt[28] = {};                        // diag view of layout A with gd = 2
    uint32_t slot_off = 0;
    uint32_t ckpt_stages = 1;      // k in stages
    uint32_t ckpt_layers = 0;      // k in layers as reported
    uint32_t ckpt_passes = 1;      // k in passes (streaming)
    uint32_t n_slots = 0;
    std::vector<qf_gate> gates;    // as given (per-gate comparator)

    bool slot_pass(size_t p) const {
        return (p + 1 + slot_off) % ckpt_passes == 0 || p + 1 == steps.size();
    }
    size_t slot_index(size_t p) const { return (p + slot_off) / ckpt_passes; }
    const PassStep &bstep(size_t p) const { return alt ? bsteps[p] : steps[p]; }
};

Plan make_plan(const qf_gate *gates, size_t n_gates, uint32_t n_qubits, uint32_t n_params,
               uint32_t layers, uint32_t ckpt_layers, uint32_t batch, uint64_t x_mask,
               uint64_t z_mask);

} // namespace qfb
