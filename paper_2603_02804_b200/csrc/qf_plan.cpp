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
#include <cstdlib>
#include <map>

namespace qfb {

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
    auto adjacency = [&](const std::vector<std::pair<uint32_t, uint32_t>> &pairs) {
        std::vector<uint32_t> adj(32, 0);
        for (auto [x, y] : pairs) { // repeated CZ pairs cancel (parity)
            adj[x] ^= 1u << y;
            adj[y] ^= 1u << x;
        }
        return adj;
    };
    std::vector<std::vector<uint32_t>> adjs;
    auto intern = [&](const std::vector<std::pair<uint32_t, uint32_t>> &pairs) {
        const auto a = adjacency(pairs);
        for (size_t k = 0; k < adjs.size(); ++k)
            if (adjs[k] == a) return static_cast<int>(k);
        adjs.push_back(a);
        plan.czsets.push_back(pairs);
        return static_cast<int>(adjs.size() - 1);
    };
    for (auto &[t, pairs] : b.cz_at) {
        if (t >= S) final_pairs.insert(final_pairs.end(), pairs.begin(), pairs.end());
        else plan.stage_cz[t] = intern(pairs);
    }
    if (!final_pairs.empty()) {
        const auto a = adjacency(final_pairs);
        CzAdj f{};
        for (int q = 0; q < 32; ++q) f.adjlo[q] = a[q] & ((1u << q) - 1u);
        plan.final_adj.push_back(f);
    }

    // ---- layouts
    plan.resident = n <= static_cast<uint32_t>(kTileBits);
    auto finish_layout = [&](PassLayout &L) {
        // diag-group view: register bits, thread bits (other local bits in order), tile bits
        for (int i = 0; i < 28; ++i) L.dq[i] = -1;
        int t = 0;
        for (int l = 0; l < 12; ++l) {
            if (l / 4 == L.gd) L.dq[l % 4] = L.qmap[l];
            else L.dq[4 + t++] = L.qmap[l];
        }
        for (size_t i = 0; i < L.tile_qubits.size() && i < 16; ++i) L.dq[12 + i] = L.tile_qubits[i];
    };
    if (plan.resident) {
        PassLayout R;
        R.row_start = 4;
        for (int l = 0; l < 12; ++l) R.qmap[l] = l < static_cast<int>(n) ? l : -1;
        R.rot_mask = (1u << std::min<uint32_t>(n, 12)) - 1u;
        R.gd = 0;
        finish_layout(R);
        plan.layouts.push_back(R);
        if (n == 12) { // chained stages (qf_resident.cu): odd stages apply D in group 2
            PassLayout R2 = R;
            R2.gd = 2;
            finish_layout(R2);
            plan.layouts.push_back(R2);
        }
    } else {
        PassLayout A;
        A.row_start = 4;
        A.tile_lo_bits = 0;
        A.tile_hi_bits = static_cast<int>(n) - 12;
        A.rot_mask = 0xFFFu;
        A.gd = 0;
        for (int l = 0; l < 12; ++l) A.qmap[l] = l;
        for (int q = 12; q < static_cast<int>(n); ++q) A.tile_qubits.push_back(q);
        finish_layout(A);
        plan.layouts.push_back(A);
        int hi = static_cast<int>(n); // qubits [12, hi) still need a layout
        while (hi > 12) {
            const int a = std::max(4, hi - 8);
            PassLayout P;
            P.row_start = a;
            P.tile_lo_bits = a - 4;
            P.tile_hi_bits = static_cast<int>(n) - a - 8;
            for (int l = 0; l < 4; ++l) P.qmap[l] = l;
            for (int l = 4; l < 12; ++l) P.qmap[l] = a + (l - 4);
            for (int l = 4; l < 12; ++l)
                if (P.qmap[l] >= 12 && P.qmap[l] < hi) P.rot_mask |= 1u << l;
            P.gd = (P.rot_mask & 0xF00u) ? 2 : 1;
            for (int q = 4; q < a; ++q) P.tile_qubits.push_back(q);
            for (int q = a + 8; q < static_cast<int>(n); ++q) P.tile_qubits.push_back(q);
            finish_layout(P);
            plan.layouts.push_back(P);
            hi = a;
        }
        // 13 <= n <= 16: layout B rotates at most 4 row qubits (one phase) while A
        // rotates 12 (five phases). Moving the column group's Ry (qubits 0..3)
        // from A to B balances them at three phases each (same total work, but
        // neither pass is left bound by one resource).
        // (The same holds for the last layout at n = 21, 22: it rotates 1-2 qubits.)
        if (plan.layouts.size() >= 2 && (plan.layouts.back().rot_mask & 0x0FFu) == 0 &&
            __builtin_popcount(plan.layouts.back().rot_mask) <= 4) {
            PassLayout &LA = plan.layouts[0], &LB = plan.layouts.back();
            LA.rot_mask = 0xFF0u;
            LA.gd = 2;
            LB.rot_mask |= 0x00Fu;
            LB.gd = 2;
            finish_layout(LA);
            finish_layout(LB);
        }
    }
    const int NL = static_cast<int>(plan.layouts.size());

    // ---- CZ sign tables per (CZ set, layout)
    auto cz_tables = [&](const std::vector<uint32_t> &adj, const PassLayout &L, CzTab &ct,
                         std::vector<uint32_t> &ti) {
        auto qset = [&](const int *qs, int k, uint32_t v) { // Q of the set bits
            uint32_t par = 0;
            for (int i = 0; i < k; ++i) {
                if (!((v >> i) & 1u) || qs[i] < 0) continue;
                for (int j = i + 1; j < k; ++j)
                    if (((v >> j) & 1u) && qs[j] >= 0) par ^= (adj[qs[i]] >> qs[j]) & 1u;
            }
            return par;
        };
        auto cross = [&](const int *qs, int k, uint32_t v, const int *to, int kto) {
            uint32_t m = 0;
            for (int i = 0; i < k; ++i) {
                if (!((v >> i) & 1u) || qs[i] < 0) continue;
                for (int r = 0; r < kto; ++r)
                    if (to[r] >= 0) m ^= ((adj[qs[i]] >> to[r]) & 1u) << r;
            }
            return m;
        };
        const int *reg = L.dq, *thr = L.dq + 4;
        ct = CzTab{};
        for (uint32_t j = 0; j < 16; ++j) ct.qreg |= qset(reg, 4, j) << j;
        for (uint32_t tau = 0; tau < 256; ++tau)
            ct.thrinfo[tau] = static_cast<uint16_t>((qset(thr, 8, tau) << 4) | cross(thr, 8, tau, reg, 4));
        const int kt = static_cast<int>(L.tile_qubits.size());
        ti.assign(size_t(1) << kt, 0u);
        for (uint32_t tb = 0; tb < ti.size(); ++tb)
            ti[tb] = qset(L.tile_qubits.data(), kt, tb) | (cross(L.tile_qubits.data(), kt, tb, reg, 4) << 1) |
                     (cross(L.tile_qubits.data(), kt, tb, thr, 8) << 8);
    };
    for (size_t c = 0; c < adjs.size(); ++c) {
        for (int li = 0; li < NL; ++li) {
            CzTab ct;
            std::vector<uint32_t> ti;
            cz_tables(adjs[c], plan.layouts[li], ct, ti);
            plan.cztab.push_back(ct);
            plan.tileinfo.push_back(std::move(ti));
        }
    }

    // ---- wide-group view of layout A (forward passes rotating all 12 local qubits)
    if (!plan.resident && plan.layouts[0].rot_mask == 0xFFFu) {
        const PassLayout &L = plan.layouts[0];
        plan.wide = true;
        for (int i = 0; i < 28; ++i) plan.dqw[i] = -1;
        for (int b = 0; b < 6; ++b) {
            plan.dqw[b] = L.qmap[wide_reg_bit(b)];
            plan.dqw[6 + b] = L.qmap[wide_thr_bit(b)];
        }
        for (size_t i = 0; i < L.tile_qubits.size() && i < 16; ++i) plan.dqw[12 + i] = L.tile_qubits[i];
        for (size_t c = 0; c < adjs.size(); ++c) {
            const auto &adj = adjs[c];
            auto qset = [&](const int *qs, int k, uint32_t v) {
                uint32_t par = 0;
                for (int i = 0; i < k; ++i) {
                    if (!((v >> i) & 1u) || qs[i] < 0) continue;
                    for (int j = i + 1; j < k; ++j)
                        if (((v >> j) & 1u) && qs[j] >= 0) par ^= (adj[qs[i]] >> qs[j]) & 1u;
                }
                return par;
            };
            auto cross = [&](const int *qs, int k, uint32_t v, const int *to, int kto) {
                uint32_t m = 0;
                for (int i = 0; i < k; ++i) {
                    if (!((v >> i) & 1u) || qs[i] < 0) continue;
                    for (int r = 0; r < kto; ++r)
                        if (to[r] >= 0) m ^= ((adj[qs[i]] >> to[r]) & 1u) << r;
                }
                return m;
            };
            const int *reg = plan.dqw, *thr = plan.dqw + 6;
            CzTabW ct{};
            for (uint32_t j = 0; j < 64; ++j) ct.qreg |= (unsigned long long)qset(reg, 6, j) << j;
            for (uint32_t tau = 0; tau < 64; ++tau)
                ct.thrinfo[tau] = static_cast<uint16_t>((qset(thr, 6, tau) << 6) | cross(thr, 6, tau, reg, 6));
            plan.cztabw.push_back(ct);
            const int kt = static_cast<int>(L.tile_qubits.size());
            std::vector<uint32_t> ti(size_t(1) << kt);
            for (uint32_t tb = 0; tb < ti.size(); ++tb)
                ti[tb] = qset(L.tile_qubits.data(), kt, tb) | (cross(L.tile_qubits.data(), kt, tb, reg, 6) << 1) |
                         (cross(L.tile_qubits.data(), kt, tb, thr, 6) << 8);
            plan.tileinfow.push_back(std::move(ti));
        }
    }

    // ---- pass sequence (streaming): a pass on layout X applies Ry_{r[X]}(X); when
    // every layout has finished stage dnext-1 it also applies D_{dnext} and, on
    // its own qubits, Ry_{dnext}. Two layouts -> one pass per stage.
    plan.stage_layout.assign(S, 0);
    if (plan.resident && n == 12)
        for (int t = 0; t < S; ++t) plan.stage_layout[t] = t & 1;
    if (!plan.resident && S > 0) {
        std::vector<int> r(NL, 0);
        int dnext = 0, X = 0;
        auto all_done = [&](int st) {
            for (int y = 0; y < NL; ++y)
                if (r[y] < st) return false;
            return true;
        };
        while (true) {
            bool finished = true;
            for (int y = 0; y < NL; ++y) finished &= r[y] >= S;
            if (finished) break;
            PassStep st;
            st.layout = X;
            if (r[X] < S && dnext > r[X]) st.s0 = r[X]++;
            if (dnext < S && all_done(dnext)) {
                st.sd = dnext;
                plan.stage_layout[dnext] = X;
                ++dnext;
                if (r[X] < S && dnext > r[X]) st.s1 = r[X]++;
            }
            // phases: round-0 groups (gd last), then round-1 groups
            // Groups 0 and 1 share their warp bits (qf_device.cuh prog_cross): the
            // round-0 group next to gd is its warp-bit partner, round 1 mirrored,
            // so the compiled programs sync those transitions with __syncwarp.
            const PassLayout &L = plan.layouts[X];
            std::vector<int> groups;
            for (int g = 0; g < 3; ++g)
                if (g != L.gd && (L.rot_mask >> (4 * g)) & 0xFu) groups.push_back(g);
            auto partner = [](int a, int b) { return a != 2 && b != 2; };
            if (groups.size() == 2 && partner(groups[0], L.gd) && !partner(groups[1], L.gd))
                std::swap(groups[0], groups[1]);
            auto add = [&](int g, uint8_t ops) { st.ph[st.nph++] = PassPhase{int8_t(g), ops}; };
            const uint8_t d_op = st.sd >= 0 ? 2 : 0;
            const uint8_t gd_ops = uint8_t((st.s0 >= 0 ? 1 : 0) | d_op | (st.s1 >= 0 ? 4 : 0));
            if (gd_ops == 1) { // round 0 only: any order; gd first, then its partner
                add(L.gd, 1);
                for (auto it = groups.rbegin(); it != groups.rend(); ++it) add(*it, 1);
            } else {
                if (st.s0 >= 0)
                    for (int g : groups) add(g, 1);
                if (gd_ops) add(L.gd, gd_ops);
                if (st.s1 >= 0)
                    for (auto it = groups.rbegin(); it != groups.rend(); ++it) add(*it, 4);
            }
            plan.steps.push_back(st);
            X = (X + 1) % NL;
        }
    }

    // checkpoint interval
    const uint32_t stages_per_layer =
        (layers > 0 && S % static_cast<int>(layers) == 0) ? static_cast<uint32_t>(S) / layers : 1u;
    uint32_t k = ckpt_layers ? ckpt_layers * stages_per_layer : std::min<uint32_t>(S ? S : 1, 10u);
    if (k == 0) k = 1;
    plan.ckpt_stages = k;
    plan.ckpt_layers = ckpt_layers ? ckpt_layers : k / std::max(1u, stages_per_layer);
    if (plan.resident) {
        const uint32_t blocks = S == 0 ? 1 : (static_cast<uint32_t>(S) + k - 1) / k;
        plan.n_slots = blocks > 0 ? blocks - 1 : 0;
    } else {
        const uint32_t pps = static_cast<uint32_t>(std::max(1, NL - 1));
        plan.ckpt_passes = k * pps;
        const size_t np = plan.steps.size();
        // balanced backward (Plan::alt): 17 <= n <= 20 with layouts A (12 rotated) and B
        // (top rows 12..n-1), strict A/B alternation with pass p applying D_p, an even
        // slot period
        const char *ea = getenv("QF_ALT");
        const uint32_t rowsB = plan.layouts.size() >= 2 ? plan.layouts[1].rot_mask : 0u;
        bool alt = (!ea || atoi(ea) != 0) && n >= 17 && n <= 20 && NL == 2 &&
                   plan.layouts[0].rot_mask == 0xFFFu && plan.layouts[0].gd == 0 &&
                   (rowsB & 0xF0Fu) == 0xF00u && (rowsB & 0x0F0u) != 0u && plan.layouts[1].gd == 2 &&
                   plan.ckpt_passes % 2 == 0 && np >= 2;
        for (size_t pi = 0; alt && pi < np; ++pi) {
            const PassStep &ps = plan.steps[pi];
            const int p = static_cast<int>(pi);
            if (pi + 1 < np)
                alt = ps.layout == p % 2 && ps.sd == p && ps.s1 == p && ps.s0 == p - 1;
            else
                alt = ps.layout == p % 2 && ps.sd < 0 && ps.s1 < 0 && ps.s0 == p - 1 && p == S;
        }
        if (alt) {
            plan.alt = true;
            plan.slot_off = 1;
            PassLayout LA = plan.layouts[0];
            LA.gd = 2;
            finish_layout(LA);
            for (int i = 0; i < 28; ++i) plan.dq_alt[i] = LA.dq[i];
            for (size_t c = 0; c < adjs.size(); ++c) {
                CzTab ct;
                std::vector<uint32_t> ti;
                cz_tables(adjs[c], LA, ct, ti);
                plan.cztab_alt.push_back(ct);
                plan.tileinfo_alt.push_back(std::move(ti));
            }
            for (const PassStep &ps : plan.steps) {
                // round 0: the layout's 8 row qubits; D; round 1: rows + columns
                PassStep b = ps;
                const uint32_t rows = ps.layout == 0 ? 0xFF0u : rowsB;
                b.rot0 = ps.s0 >= 0 ? rows : 0u;
                b.rot1 = ps.s1 >= 0 ? (rows | 0x00Fu) : 0u;
                b.nph = 0;
                auto add = [&](int g, uint8_t ops) { b.ph[b.nph++] = PassPhase{int8_t(g), ops}; };
                const uint8_t gd_ops = uint8_t((ps.s0 >= 0 ? 1 : 0) | (ps.sd >= 0 ? 2 : 0) | (ps.s1 >= 0 ? 4 : 0));
                if (ps.s0 >= 0) add(1, 1);
                add(2, gd_ops);
                if (ps.s1 >= 0) {
                    add(1, 4);
                    add(0, 4);
                }
                plan.bsteps.push_back(b);
            }
        }
        plan.n_slots = np == 0 ? 0 : static_cast<uint32_t>((np - 1 + plan.slot_off) / plan.ckpt_passes + 1);
    }
    return plan;
}

} // namespace qfb
