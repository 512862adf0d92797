// Host planner (theta-independent).
//
// Input is the reference's flattened gate IR (fusion.cpp:103-125; HEA order
// circuit.cpp:89-114). Every maximal run of single-qubit gates on a qubit
// (a *section*) becomes U = e^{i d} Rz(a) Ry(b) Rz(g) at device time; the
// planner only decides WHERE things go:
//   * the section's Ry(b) goes to stage s = max(q's previous stage + 1,
//     stage of the last CZ touching q);
//   * Rz(g) joins the diagonal of stage s, Rz(a) the diagonal of q's next
//     section's stage (or the final diagonal);
//   * CZ(a, b) joins the diagonal of stage max(last Ry of a, b) + 1;
//   * CNOT(c, t) = H_t CZ(c, t) H_t with H = Ry(pi/2) Z, so it is expressed with
//     a fixed H inside t's sections.
// Diagonals commute, so every constraint is "after the previous Ry of the
// same qubit, before its next one". For the HEA this yields exactly one stage
// per layer.
#include "qf_plan.h"

#include <algorithm>
#include <map>

namespace qfb {

CzSet make_czset(const std::vector<std::pair<uint32_t, uint32_t>> &pairs) {
    CzSet c{};
    for (auto [a, b] : pairs) { // repeated CZ pairs cancel (parity)
        c.adj[a] ^= 1u << b;
        c.adj[b] ^= 1u << a;
    }
    for (int q = 0; q < 32; ++q) c.adjlo[q] = c.adj[q] & ((1u << q) - 1u);
    auto qform = [&](uint32_t v) {
        uint32_t par = 0;
        for (int q = 0; q < 32; ++q)
            if ((v >> q) & 1u) par ^= __builtin_popcount(v & c.adjlo[q]);
        return par & 1u;
    };
    c.qcol = 0;
    for (uint32_t j = 0; j < 16; ++j) c.qcol |= qform(j) << j;
    for (uint32_t r = 0; r < 256; ++r) {
        const uint32_t v = r << 4;
        uint32_t m = 0;
        for (int q = 4; q < 12; ++q)
            if ((v >> q) & 1u) m ^= c.adj[q] & 15u;
        c.rowinfo[r] = static_cast<uint8_t>((qform(v) << 4) | m);
    }
    return c;
}

namespace {

struct Builder {
    uint32_t n;
    std::vector<std::vector<uint32_t>> pending;
    std::vector<int> last_ry, min_stage, last_sec;
    std::map<int, std::vector<std::pair<uint32_t, uint32_t>>> cz_at;
    int n_stages = 0;
    Plan &plan;

    Builder(uint32_t n_, Plan &p)
        : n(n_), pending(n_), last_ry(n_, -1), min_stage(n_, 0), last_sec(n_, -1), plan(p) {}

    void flush(uint32_t q) {
        if (pending[q].empty()) return;
        const int s = std::max(min_stage[q], last_ry[q] + 1);
        n_stages = std::max(n_stages, s + 1);
        const auto idx = static_cast<int>(plan.sec_q.size());
        plan.sec_q.push_back(q);
        plan.sec_stage.push_back(static_cast<uint32_t>(s));
        plan.sec_alpha_row.push_back(0); // fixed when q's next section (or the end) is known
        plan.sec_off.push_back(static_cast<uint32_t>(plan.sec_gates.size()));
        plan.sec_gates.insert(plan.sec_gates.end(), pending[q].begin(), pending[q].end());
        if (last_sec[q] >= 0) plan.sec_alpha_row[last_sec[q]] = static_cast<uint32_t>(s);
        last_sec[q] = idx;
        last_ry[q] = s;
        pending[q].clear();
    }
    void cz(uint32_t a, uint32_t b) {
        flush(a);
        flush(b);
        const int t = std::max(last_ry[a], last_ry[b]) + 1;
        cz_at[t].emplace_back(a, b);
        min_stage[a] = std::max(min_stage[a], t);
        min_stage[b] = std::max(min_stage[b], t);
    }
};

void invalid(const std::string &m) { throw std::invalid_argument(m); }

} // namespace

Plan make_plan(const qf_gate *gates, size_t n_gates, uint32_t n, uint32_t n_params,
               uint32_t layers, uint32_t ckpt_layers, uint32_t batch, uint64_t x_mask,
               uint64_t z_mask) {
    // ---- validation, mirroring the reference's constructors
    if (n == 0) invalid("BatchedState: qubit count must be >= 1");          // statevec.hpp:84-86
    if (batch == 0) invalid("BatchedState: batch must be >= 1");           // statevec.hpp:87-89
    if (n > static_cast<uint32_t>(kMaxQubits))
        throw CapacityError("BatchedState: qubit count above supported range"); // :89-91
    if (gates == nullptr && n_gates != 0) invalid("gradient: null gate list");
    std::vector<uint32_t> uses(n_params, 0);
    for (size_t i = 0; i < n_gates; ++i) { // Circuit::Circuit, circuit.cpp:27-59
        const qf_gate &g = gates[i];
        if (g.kind == QF_GATE_ROTATION) {
            if (g.axis > QF_AXIS_Z) invalid("Circuit: unknown rotation axis");
            if (g.q0 >= n) invalid("Circuit: rotation target out of range");
            if (g.param >= n_params) invalid("Circuit: parameter index out of range");
            ++uses[g.param];
        } else if (g.kind == QF_GATE_CZ || g.kind == QF_GATE_CNOT) {
            if (g.q0 >= n || g.q1 >= n) invalid("Circuit: two-qubit gate out of range");
            if (g.q0 == g.q1) invalid("Circuit: control equals target");
        } else {
            invalid("Circuit: unknown gate kind");
        }
    }
    for (uint32_t j = 0; j < n_params; ++j)
        if (uses[j] != 1)
            invalid("Circuit: parameter " + std::to_string(j) + " used " + std::to_string(uses[j]) +
                    " times (expected exactly once)");
    const uint64_t width = n >= 64 ? ~0ull : ((1ull << n) - 1);
    if ((x_mask & ~width) || (z_mask & ~width))
        invalid("PauliString: mask wider than qubit count"); // circuit.cpp:150-154
    if (ckpt_layers != 0) { // CheckpointPlan::uniform, checkpoint.cpp:24-49
        if (layers == 0) invalid("checkpoint: layer counts must be positive");
        if (layers % ckpt_layers != 0)
            invalid("checkpoint: block size " + std::to_string(ckpt_layers) +
                    " does not divide layer count " + std::to_string(layers));
        if (n_gates == 0 || n_gates % layers != 0)
            invalid("checkpoint: op count is not layer-periodic");
    }

    Plan plan;
    plan.n = n;
    plan.n_params = n_params;
    plan.layers = layers;
    plan.batch = batch;
    plan.x_mask = x_mask;
    plan.z_mask = z_mask;
    plan.y_count = static_cast<uint32_t>(__builtin_popcountll(x_mask & z_mask));
    plan.gates.assign(gates, gates + n_gates);

    // ---- sections and stages
    Builder b(n, plan);
    for (size_t i = 0; i < n_gates; ++i) {
        const qf_gate &g = gates[i];
        if (g.kind == QF_GATE_ROTATION) {
            b.pending[g.q0].push_back(uint32_t(g.axis) | (g.param << 2));
        } else if (g.kind == QF_GATE_CZ) {
            b.cz(g.q0, g.q1);
        } else { // CNOT(c, t) = H_t CZ(c, t) H_t
            b.pending[g.q1].push_back(kSecH);
            b.cz(g.q0, g.q1);
            b.pending[g.q1].push_back(kSecH);
        }
    }
    for (uint32_t q = 0; q < n; ++q) b.flush(q);
    const int S = b.n_stages;
    plan.stages = static_cast<uint32_t>(S);
    for (uint32_t q = 0; q < n; ++q)
        if (b.last_sec[q] >= 0) plan.sec_alpha_row[b.last_sec[q]] = static_cast<uint32_t>(S);
    plan.sec_off.push_back(static_cast<uint32_t>(plan.sec_gates.size()));

    // CZ sets per stage (deduplicated) and the final one
    plan.stage_cz.assign(S, -1);
    std::vector<std::pair<uint32_t, uint32_t>> final_pairs;
    auto intern = [&](const std::vector<std::pair<uint32_t, uint32_t>> &pairs) {
        const CzSet c = make_czset(pairs);
        for (size_t k = 0; k < plan.czsets.size(); ++k)
            if (std::equal(std::begin(c.adj), std::end(c.adj), std::begin(plan.czsets[k].adj)))
                return static_cast<int>(k);
        plan.czsets.push_back(c);
        return static_cast<int>(plan.czsets.size() - 1);
    };
    for (auto &[t, pairs] : b.cz_at) {
        if (t >= S) final_pairs.insert(final_pairs.end(), pairs.begin(), pairs.end());
        else plan.stage_cz[t] = intern(pairs);
    }
    if (!final_pairs.empty()) plan.final_cz = intern(final_pairs);

    // ---- schedule
    plan.resident = n <= static_cast<uint32_t>(kTileBits);
    if (!plan.resident) {
        PassLayout A{};
        A.row_start = 4;
        A.tile_lo_bits = 0;
        A.tile_hi_bits = static_cast<int>(n) - 12;
        A.rot_mask = 0xFFFu;
        A.has_diag = true;
        for (int l = 0; l < 12; ++l) A.qmap[l] = l;
        plan.passes.push_back(A);
        // remaining qubits 12..n-1 in 8-row blocks from the top
        int hi = static_cast<int>(n); // rotate [lo, hi)
        while (hi > 12) {
            const int a = std::max(4, hi - 8);
            PassLayout P{};
            P.row_start = a;
            P.tile_lo_bits = a - 4;
            P.tile_hi_bits = static_cast<int>(n) - a - 8;
            P.has_diag = false;
            for (int l = 0; l < 4; ++l) P.qmap[l] = l;
            for (int l = 4; l < 12; ++l) P.qmap[l] = a + (l - 4);
            P.rot_mask = 0;
            for (int l = 4; l < 12; ++l)
                if (P.qmap[l] >= 12 && P.qmap[l] < hi) P.rot_mask |= 1u << l;
            plan.passes.push_back(P);
            hi = a;
        }
    }
    // checkpoint interval in stages
    const uint32_t stages_per_layer =
        (layers > 0 && S % static_cast<int>(layers) == 0) ? static_cast<uint32_t>(S) / layers : 1u;
    uint32_t k = ckpt_layers ? ckpt_layers * stages_per_layer : std::min<uint32_t>(S ? S : 1, 10u);
    if (k == 0) k = 1;
    plan.ckpt_stages = k;
    plan.ckpt_layers = ckpt_layers ? ckpt_layers : k / std::max(1u, stages_per_layer);
    const uint32_t blocks = S == 0 ? 1 : (static_cast<uint32_t>(S) + k - 1) / k;
    plan.n_slots = plan.resident ? (blocks > 0 ? blocks - 1 : 0) : blocks;
    return plan;
}

} // namespace qfb
