// C-ABI of qfuse-b200 (include/qfuse_b200.h): device store, checkpoint
// slots, the fused schedule and the per-gate comparator.
//
// Schedule U: the forward runs every stage's passes in place
// on one working buffer and lands the last pass of every k-th stage in a
// checkpoint slot; the backward uncomputes psi with the inverse stages and
// re-anchors it from the slot at each block end, so the backward never
// stores an intermediate state (the reference instead replays each block
// into a ledger, checkpoint.cpp:123-135; both give the same gradients).
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/qfuse_b200.h"
#include "qf_internal.h"
#include "qf_plan.h"

using namespace qfb;

namespace {

thread_local std::string g_err;

struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char *what) {
    if (e != cudaSuccess)
        throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F> int guarded(F &&f) {
    try {
        f();
        return QF_OK;
    } catch (const CapacityError &e) {
        g_err = e.what();
        return QF_ECAPACITY;
    } catch (const std::invalid_argument &e) {
        g_err = e.what();
        return QF_EINVAL;
    } catch (const std::bad_alloc &e) {
        g_err = "host allocation failed";
        return QF_ECAPACITY;
    } catch (const std::exception &e) {
        g_err = e.what();
        return QF_EDEVICE;
    }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                   const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                   const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    if (!fn) throw DeviceError("cuTensorMapEncodeTiled unavailable");
    return fn;
}

CUtensorMap encode(void *base, int rank, const cuuint64_t *dims, const cuuint64_t *strides,
                   const cuuint32_t *box) {
    CUtensorMap m;
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, base, dims, strides,
                                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw DeviceError("cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

// 5-D view of a batch store for a streaming pass (see qf_internal.h).
CUtensorMap pass_map(void *base, const PassLayout &L, uint32_t n, uint32_t batch) {
    const int a = L.row_start;
    cuuint64_t dims[5] = {32, 1ull << L.tile_lo_bits, 256, 1ull << L.tile_hi_bits, batch};
    cuuint64_t strides[4] = {128, 8ull << a, 8ull << (a + 8), 8ull << n};
    cuuint32_t box[5] = {32, 1, 256, 1, 1};
    return encode(base, 5, dims, strides, box);
}
// 3-D view [buffers][rows][32 floats] for the resident kernel.
CUtensorMap flat_map(void *base, uint64_t rows, uint64_t nbuf, uint64_t buf_bytes) {
    cuuint64_t dims[3] = {32, rows, nbuf ? nbuf : 1};
    cuuint64_t strides[2] = {128, buf_bytes};
    cuuint32_t box[3] = {32, 256, 1};
    return encode(base, 3, dims, strides, box);
}

// NVTX range around the host enqueue of one phase of a gradient (forward passes,
// observable, backward passes, reductions): `ncu --nvtx --nvtx-include
// "qfuse backward/"` selects one phase's kernels. Header-only NVTX: a no-op
// unless a tool is attached.
struct Nvtx {
    explicit Nvtx(const char *name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx &) = delete;
    Nvtx &operator=(const Nvtx &) = delete;
};

template <class T> T *dalloc(size_t count, std::vector<void *> &owned) {
    if (count == 0) count = 1;
    void *p = nullptr;
    const cudaError_t e = cudaMalloc(&p, count * sizeof(T));
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw CapacityError("device allocation of " + std::to_string(count * sizeof(T)) +
                            " bytes failed: " + cudaGetErrorString(e));
    }
    owned.push_back(p);
    return static_cast<T *>(p);
}
template <class T> T *dupload(const std::vector<T> &v, std::vector<void *> &owned) {
    T *p = dalloc<T>(v.size(), owned);
    if (!v.empty()) ck(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
    return p;
}

} // namespace

struct qf_ctx {
    int device = 0;
    int sms = 148;
    uint64_t hbm_limit = 0;
    cudaStream_t stream = nullptr;
    // One-shot entry points (qf_gradient_c64*, the reference-signature calls): the
    // last plan is kept and reused while the next call has the same circuit, shape
    // and storage mode (a training loop calls gradient<float> with new theta and
    // psi0 every step, bench.cpp:114-133), so a call costs its H2D + the gradient,
    // not a plan build. Explicit plan creation on the context drops it first.
    qf_plan *cached = nullptr;
    std::string cache_key;
    bool cache_enabled = true;
    // pinned staging of host psi0 for the one-shot calls (filled by host threads,
    // DMA'd chunk by chunk while the next chunks are still being copied)
    float *stage = nullptr;
    size_t stage_bytes = 0;
};

struct qf_plan {
    qf_ctx *ctx = nullptr;
    Plan P;
    std::vector<void *> owned;
    uint64_t amps = 0;        // B * 2^n
    uint64_t amps_padded = 0; // multiple of one tile
    size_t state_bytes = 0;
    // stores. psi0 is the plan's own input buffer; psi0_src is where the passes read
    // psi0 from (psi0, or caller memory bound by qf_plan_set_psi0_device)
    float2 *psi0 = nullptr, *W = nullptr, *lam = nullptr, *slots = nullptr;
    const float2 *psi0_src = nullptr;
    // StorageMode::MemSave (streaming plans): checkpoint slots as bfloat16 pairs,
    // the final state stays complex64 in W
    uint32_t storage = QF_STORAGE_FULL;
    uint32_t *slots16 = nullptr;
    uint64_t device_bytes = 0; // batch store + slots + K partials
    bool memsave() const { return storage == QF_STORAGE_MEMSAVE && !P.resident; }
    // theta-dependent stage data
    double *theta = nullptr, *out = nullptr;
    float2 *ry = nullptr;
    DiagTab *dtab = nullptr;
    DiagTabW *dtabw = nullptr; // wide-group tables (layout 0), nullptr when !P.wide
    CzTabW *cztabw = nullptr;
    uint32_t *tileinfow = nullptr;
    std::vector<size_t> tileinfow_off; // [czset]
    int *dqw = nullptr;
    double *wg = nullptr, *wa = nullptr, *wfinal = nullptr, *sec_gamma = nullptr, *sec_phase = nullptr;
    // theta-independent tables
    CzTab *cztab = nullptr;
    uint32_t *tileinfo = nullptr;
    std::vector<size_t> tileinfo_off; // [czset * layouts + layout]
    CzAdj *final_adj = nullptr;
    int *stage_cz = nullptr, *stage_layout = nullptr, *dq = nullptr;
    // balanced backward (P.alt): diagonal tables of layout A in the group-2 view
    DiagTab *dtab_alt = nullptr;
    CzTab *cztab_alt = nullptr;
    uint32_t *tileinfo_alt = nullptr;
    std::vector<size_t> tileinfo_alt_off; // [czset]
    int *dq_alt = nullptr;                // [A with gd = 2, B][28]
    uint32_t *sec_q = nullptr, *sec_stage = nullptr, *sec_alpha = nullptr, *sec_off = nullptr,
             *sec_gates = nullptr;
    double *kpart = nullptr, *kout = nullptr, *epart = nullptr;
    int grid_fwd = 0, grid_bwd = 0, grid_res = 0;
    // tensor maps
    std::vector<CUtensorMap> m_psi0, m_W, m_lam; // per layout
    std::vector<std::vector<CUtensorMap>> m_slot; // [slot][layout]
    CUtensorMap r_psi0{}, r_slots{}, r_out{};
    // per-gate comparator
    double *gpart = nullptr;
    uint32_t *rot_params = nullptr;
    int n_rot = 0, gblocks = 0;
    // host staging
    double *h_theta = nullptr, *h_out = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    qf_stats last{};
    // per-launch CUDA-event profiling (qf_plan_set_profiling)
    bool profiling = false;
    std::vector<cudaEvent_t> ev_pool;
    struct Mark {
        int kind;
        size_t e0, e1;
        double bytes;
    };
    std::vector<Mark> marks;
    size_t ev_used = 0;
    double prof_ms[8] = {}, prof_bytes[8] = {};
    uint64_t prof_launches[8] = {};
    double *rand_scratch = nullptr;

    size_t record() {
        if (ev_used == ev_pool.size()) {
            cudaEvent_t e;
            ck(cudaEventCreate(&e), "event");
            ev_pool.push_back(e);
        }
        ck(cudaEventRecord(ev_pool[ev_used], ctx->stream), "event record");
        return ev_used++;
    }
    // Wraps one launch; kind: 0 fwd pass, 1 bwd pass, 2 observable, 3 resident,
    // 4 prep/reduce/finalize, 5 per-gate.
    template <class F> void timed(int kind, double bytes, F &&launch) {
        if (!profiling) {
            launch();
            return;
        }
        const size_t a = record();
        launch();
        const size_t b = record();
        marks.push_back({kind, a, b, bytes});
    }
    void harvest() {
        if (marks.empty()) return;
        ck(cudaStreamSynchronize(ctx->stream), "profile sync");
        for (const Mark &m : marks) {
            float ms = 0;
            ck(cudaEventElapsedTime(&ms, ev_pool[m.e0], ev_pool[m.e1]), "elapsed");
            prof_ms[m.kind] += ms;
            prof_bytes[m.kind] += m.bytes;
            prof_launches[m.kind]++;
        }
        marks.clear();
        ev_used = 0;
    }

    ~qf_plan() {
        if (ctx) cudaSetDevice(ctx->device);
        for (void *p : owned) cudaFree(p);
        if (h_theta) cudaFreeHost(h_theta);
        if (h_out) cudaFreeHost(h_out);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
    }
    size_t out_len() const { return size_t(P.n_params) + 1 + P.batch; }
    const uint32_t *tinfo(int cz, int layout) const {
        return tileinfo + tileinfo_off[size_t(cz) * P.layouts.size() + layout];
    }
};

namespace {

void build_device_plan(qf_plan *pl) {
    const Plan &P = pl->P;
    qf_ctx *ctx = pl->ctx;
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    pl->amps = uint64_t(P.batch) << P.n;
    pl->amps_padded = (pl->amps + kTileAmps - 1) / kTileAmps * kTileAmps;
    pl->state_bytes = size_t(pl->amps_padded) * 8;
    const uint32_t S = P.stages, n = P.n;

    // ---- capacity check before touching the allocator (CapacityError as the reference)
    const int occ_f = pass_occupancy(false), occ_b = pass_occupancy(true), occ_r = resident_occupancy();
    if (occ_f <= 0 || occ_b <= 0 || occ_r <= 0) throw DeviceError("kernel occupancy query failed");
    pl->grid_fwd = occ_f * ctx->sms;
    pl->grid_bwd = occ_b * ctx->sms;
    const uint64_t tiles_res = pl->amps_padded / kTileAmps;
    pl->grid_res = int(std::min<uint64_t>(tiles_res, uint64_t(occ_r) * ctx->sms));
    const int grid_k = P.resident ? pl->grid_res : pl->grid_bwd;
    // MemSave: slots hold bfloat16 pairs (half a state each); the last slot is
    // the final state, kept complex64 in W
    const size_t n_slot16 = pl->memsave() && P.n_slots > 0 ? P.n_slots - 1 : 0;
    const size_t n_states = P.resident ? (2 + P.n_slots) : pl->memsave() ? 3 : (3 + P.n_slots);
    const size_t kpart_bytes = size_t(grid_k) * S * n * 8 * 8;
    const size_t need = n_states * pl->state_bytes + n_slot16 * (pl->state_bytes / 2) + kpart_bytes +
                        size_t(S) * sizeof(DiagTab) + (size_t(64) << 20);
    size_t free_b = 0, total_b = 0;
    ck(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
    const uint64_t budget = ctx->hbm_limit ? std::min<uint64_t>(ctx->hbm_limit, free_b) : free_b;
    pl->device_bytes = need - (size_t(64) << 20);
    if (need > budget)
        throw CapacityError("device working set of " + std::to_string(need >> 20) +
                            " MiB (states + " + std::to_string(P.n_slots) +
                            " checkpoint slots) exceeds the HBM budget of " +
                            std::to_string(budget >> 20) + " MiB");

    auto &o = pl->owned;
    pl->psi0 = dalloc<float2>(pl->amps_padded, o);
    pl->psi0_src = pl->psi0;
    ck(cudaMemset(pl->psi0, 0, pl->state_bytes), "memset");
    pl->lam = dalloc<float2>(pl->amps_padded, o);
    if (!P.resident) pl->W = dalloc<float2>(pl->amps_padded, o);
    if (pl->memsave()) {
        pl->slots = nullptr;
        pl->slots16 = dalloc<uint32_t>(size_t(pl->amps_padded) * std::max<size_t>(1, n_slot16), o);
    } else {
        pl->slots = dalloc<float2>(size_t(pl->amps_padded) * std::max<uint32_t>(1, P.n_slots), o);
    }
    pl->theta = dalloc<double>(P.n_params, o);
    pl->out = dalloc<double>(pl->out_len(), o);
    // stage data; ry defaults to identity, w to zero (entries no section writes)
    std::vector<float2> ry_init(size_t(std::max<uint32_t>(S, 1)) * n, make_float2(1.f, 0.f));
    pl->ry = dupload(ry_init, o);
    pl->wg = dalloc<double>(size_t(S + 1) * n, o);
    pl->wa = dalloc<double>(size_t(S + 1) * n, o);
    ck(cudaMemset(pl->wg, 0, size_t(S + 1) * n * 8), "memset");
    ck(cudaMemset(pl->wa, 0, size_t(S + 1) * n * 8), "memset");
    pl->wfinal = dalloc<double>(n + 1, o); // [n]: global phase (forward-state readout)
    ck(cudaMemset(pl->wfinal, 0, (n + 1) * sizeof(double)), "memset");
    pl->dtab = dalloc<DiagTab>(std::max<uint32_t>(S, 1), o);
    if (P.wide) {
        pl->dtabw = dalloc<DiagTabW>(std::max<uint32_t>(S, 1), o);
        pl->cztabw = P.cztabw.empty() ? nullptr : dupload(P.cztabw, o);
        std::vector<uint32_t> tw;
        for (const auto &t : P.tileinfow) {
            pl->tileinfow_off.push_back(tw.size());
            tw.insert(tw.end(), t.begin(), t.end());
        }
        pl->tileinfow = tw.empty() ? nullptr : dupload(tw, o);
        pl->dqw = dupload(std::vector<int>(P.dqw, P.dqw + 28), o);
    }
    pl->sec_gamma = dalloc<double>(P.sec_q.size(), o);
    pl->sec_phase = dalloc<double>(P.sec_q.size(), o);
    pl->cztab = dupload(P.cztab, o);
    std::vector<uint32_t> ti_all;
    for (const auto &t : P.tileinfo) {
        pl->tileinfo_off.push_back(ti_all.size());
        ti_all.insert(ti_all.end(), t.begin(), t.end());
    }
    pl->tileinfo = dupload(ti_all, o);
    pl->final_adj = P.final_adj.empty() ? nullptr : dupload(P.final_adj, o);
    pl->stage_cz = dupload(P.stage_cz, o);
    pl->stage_layout = dupload(P.stage_layout, o);
    std::vector<int> dq;
    for (const PassLayout &L : P.layouts) dq.insert(dq.end(), L.dq, L.dq + 28);
    pl->dq = dupload(dq, o);
    if (P.alt) {
        pl->dtab_alt = dalloc<DiagTab>(std::max<uint32_t>(S, 1), o);
        if (!P.cztab_alt.empty()) pl->cztab_alt = dupload(P.cztab_alt, o);
        std::vector<uint32_t> ta;
        for (const auto &t : P.tileinfo_alt) {
            pl->tileinfo_alt_off.push_back(ta.size());
            ta.insert(ta.end(), t.begin(), t.end());
        }
        if (!ta.empty()) pl->tileinfo_alt = dupload(ta, o);
        std::vector<int> dqa(P.dq_alt, P.dq_alt + 28);
        dqa.insert(dqa.end(), P.layouts[1].dq, P.layouts[1].dq + 28);
        pl->dq_alt = dupload(dqa, o);
    }
    pl->sec_q = dupload(P.sec_q, o);
    pl->sec_stage = dupload(P.sec_stage, o);
    pl->sec_alpha = dupload(P.sec_alpha_row, o);
    pl->sec_off = dupload(P.sec_off, o);
    pl->sec_gates = dupload(P.sec_gates, o);
    pl->kpart = dalloc<double>(size_t(grid_k) * S * n * 8, o);
    pl->kout = dalloc<double>(size_t(S) * n * 8, o);
    const uint64_t chunks = (1ull << n) >= uint64_t(kTileAmps) ? (1ull << n) / kTileAmps : 1;
    pl->epart = dalloc<double>(size_t(P.batch) * chunks, o);

    // ---- tensor maps
    if (P.resident) {
        const uint64_t rows = pl->amps_padded / 16;
        pl->r_psi0 = flat_map(pl->psi0, rows, 1, pl->state_bytes);
        // (bind_psi0 re-encodes r_psi0 / m_psi0 for caller memory)
        pl->r_slots = flat_map(pl->slots, rows, std::max<uint32_t>(1, P.n_slots), pl->state_bytes);
        pl->r_out = flat_map(pl->lam, rows, 1, pl->state_bytes);
    } else {
        for (const PassLayout &L : P.layouts) {
            pl->m_psi0.push_back(pass_map(pl->psi0, L, n, P.batch));
            pl->m_W.push_back(pass_map(pl->W, L, n, P.batch));
            pl->m_lam.push_back(pass_map(pl->lam, L, n, P.batch));
        }
        pl->m_slot.resize(pl->memsave() ? 0 : P.n_slots);
        for (uint32_t j = 0; j < pl->m_slot.size(); ++j)
            for (const PassLayout &L : P.layouts)
                pl->m_slot[j].push_back(pass_map(pl->slots + size_t(j) * pl->amps_padded, L, n, P.batch));
    }
    // per-gate comparator bookkeeping
    std::vector<uint32_t> rp;
    for (const qf_gate &g : P.gates)
        if (g.kind == QF_GATE_ROTATION) rp.push_back(g.param);
    pl->n_rot = int(rp.size());
    pl->rot_params = dupload(rp, o);
    pl->gblocks = gate_grid(std::max<uint64_t>(1, pl->amps / 2));
    ck(cudaMallocHost(&pl->h_theta, sizeof(double) * std::max<uint32_t>(1, P.n_params)), "host alloc");
    ck(cudaMallocHost(&pl->h_out, sizeof(double) * pl->out_len()), "host alloc");
    ck(cudaEventCreate(&pl->ev0), "event");
    ck(cudaEventCreate(&pl->ev1), "event");
    ck(cudaDeviceSynchronize(), "plan setup");
}

// Points the passes' psi0 maps at `src` (the plan's own buffer or caller memory
// of batch * 2^n complex64). TMA reads rows of 128 B: caller memory must be
// 16-B aligned and cover whole rows (batch * 2^n a multiple of 16 amplitudes).
void bind_psi0(qf_plan *pl, const float2 *src) {
    if (src == pl->psi0_src) return;
    const Plan &P = pl->P;
    if (src != pl->psi0) {
        if (reinterpret_cast<uintptr_t>(src) & 15u)
            throw std::invalid_argument("qf_plan_set_psi0_device: pointer must be 16-byte aligned");
        if (pl->amps % 16u)
            throw std::invalid_argument("qf_plan_set_psi0_device: batch * 2^n must be a multiple of 16");
    }
    void *base = const_cast<float2 *>(src);
    if (P.resident) {
        // rows of the caller's buffer only; TMA fills the padded tail with zeros
        const uint64_t rows = src == pl->psi0 ? pl->amps_padded / 16 : pl->amps / 16;
        pl->r_psi0 = flat_map(base, rows, 1, pl->state_bytes);
    } else {
        for (size_t i = 0; i < P.layouts.size(); ++i) pl->m_psi0[i] = pass_map(base, P.layouts[i], P.n, P.batch);
    }
    pl->psi0_src = src;
}

// ---- the fused gradient, enqueued on the context stream
void enqueue_prep(qf_plan *pl, const double *theta_dev, qf_stats &st) {
    const Plan &P = pl->P;
    cudaStream_t s = pl->ctx->stream;
    pl->timed(4, 0, [&] {
        ck(launch_prep_sections(s, int(P.sec_q.size()), pl->sec_q, pl->sec_stage, pl->sec_alpha,
                                pl->sec_off, pl->sec_gates, theta_dev, int(P.n), pl->ry, pl->wg,
                                pl->wa, pl->sec_gamma, pl->sec_phase),
           "prep_sections");
        ck(launch_diag_tables(s, int(P.stages), int(P.n), pl->wg, pl->wa, pl->stage_layout, pl->dq,
                              pl->dtab, pl->wfinal),
           "diag_tables");
        if (P.alt)
            ck(launch_diag_tables(s, int(P.stages), int(P.n), pl->wg, pl->wa, pl->stage_layout, pl->dq_alt,
                                  pl->dtab_alt, pl->wfinal),
               "diag_tables (balanced backward)");
        if (P.wide)
            ck(launch_diag_tables_wide(s, int(P.stages), int(P.n), pl->wg, pl->wa, pl->stage_layout, pl->dqw,
                                       pl->dtabw),
               "diag_tables_wide");
    });
    st.kernel_launches += 2;
}

PassParams pass_params(qf_plan *pl, const PassStep &ps, bool write_psi, bool balanced = false) {
    const Plan &P = pl->P;
    const PassLayout &L = P.layouts[ps.layout];
    PassParams p{};
    p.n = int(P.n);
    p.tiles = int(uint64_t(P.batch) << (P.n - 12));
    p.tile_lo_bits = L.tile_lo_bits;
    p.tile_hi_bits = L.tile_hi_bits;
    p.rot0 = ps.rot0 | ps.rot1 ? ps.rot0 : L.rot_mask;
    p.rot1 = ps.rot0 | ps.rot1 ? ps.rot1 : L.rot_mask;
    p.rot_mask = p.rot0 | p.rot1;
    for (int l = 0; l < 12; ++l) p.qmap[l] = L.qmap[l];
    p.s0 = ps.s0;
    p.s1 = ps.s1;
    p.nph = ps.nph;
    for (int i = 0; i < ps.nph; ++i) p.ph[i] = ps.ph[i];
    p.gd = L.gd;
    p.ry = pl->ry;
    if (ps.sd >= 0 && balanced) { // layout A with the diagonal in group 2; layout B as is
        p.gd = 2;
        p.dt = pl->dtab_alt + ps.sd;
        const int c = P.stage_cz[ps.sd];
        if (c >= 0 && ps.layout == 0) {
            p.cz = pl->cztab_alt + c;
            p.tileinfo = pl->tileinfo_alt + pl->tileinfo_alt_off[c];
        } else if (c >= 0) {
            p.cz = pl->cztab + size_t(c) * P.layouts.size() + ps.layout;
            p.tileinfo = pl->tinfo(c, ps.layout);
        }
    } else if (ps.sd >= 0) {
        p.dt = pl->dtab + ps.sd;
        const int c = P.stage_cz[ps.sd];
        p.cz = c >= 0 ? pl->cztab + size_t(c) * P.layouts.size() + ps.layout : nullptr;
        p.tileinfo = c >= 0 ? pl->tinfo(c, ps.layout) : nullptr;
    }
    if (P.wide && ps.layout == 0 && ps.sd >= 0 && !balanced) {
        p.dtw = pl->dtabw + ps.sd;
        const int c = P.stage_cz[ps.sd];
        p.czw = c >= 0 ? pl->cztabw + c : nullptr;
        p.tileinfow = c >= 0 ? pl->tileinfow + pl->tileinfow_off[c] : nullptr;
    }
    p.write_psi = write_psi ? 1 : 0;
    p.zmask = (ps.s0 == 0 ? 1 : 0) | (ps.s1 == 0 ? 2 : 0);
    p.prog = prog_encode(p.nph, p.ph, p.rot_mask);
    static const int l2pf = [] {
        const char *e = getenv("QF_L2PF");
        return e ? atoi(e) : 1;
    }();
    p.l2pf = l2pf;
    static const int wrefill = [] { // wide forward: refill at the next tile's start (2) or at its
        const char *e = getenv("QF_WREFILL"); // first phase boundary (0, measured faster)
        return e ? atoi(e) : 0;
    }();
    if (p.dtw) p.l2pf = (p.l2pf & 1) | wrefill;
    p.kpart = pl->kpart;
    p.kstride = (long long)P.stages * P.n * 8;
    return p;
}

void enqueue_fused(qf_plan *pl, const double *theta_dev, double *out_dev, qf_stats &st,
                   bool forward_only = false) {
    const Plan &P = pl->P;
    cudaStream_t s = pl->ctx->stream;
    const uint32_t S = P.stages, n = P.n;
    enqueue_prep(pl, theta_dev, st);
    if (forward_only)
        ck(launch_phase_sum(s, int(P.sec_q.size()), pl->sec_phase, int(n), pl->wfinal), "phase sum");
    const double sb = double(pl->amps) * 8.0; // algorithmic bytes of one state
    double bytes = 0.0;
    if (P.resident) {
        if (!forward_only)
            ck(cudaMemsetAsync(pl->kpart, 0, size_t(pl->grid_res) * S * n * 8 * 8, s), "memset");
        ResidentParams r{};
        r.n = int(n);
        r.stages = int(S);
        r.ckpt = int(P.ckpt_stages);
        r.tiles = int(pl->amps_padded / kTileAmps);
        r.batch = P.batch;
        r.x_mask = P.x_mask;
        r.z_mask = P.z_mask;
        r.y_count = P.y_count;
        r.ry = pl->ry;
        r.dt = pl->dtab;
        r.cztabs = pl->cztab;
        r.cz_stride = int(P.layouts.size());
        r.stage_cz = pl->stage_cz;
        r.wfinal = pl->wfinal;
        r.czfinal = pl->final_adj;
        r.kpart = pl->kpart;
        r.expect = out_dev + P.n_params + 1;
        r.forward_only = forward_only ? 1 : 0;
        const double rb = sb * (1.0 + (forward_only ? 1.0 : 2.0 * P.n_slots));
        pl->timed(3, rb, [&] {
            ck(launch_resident(s, pl->grid_res, r, &pl->r_psi0, &pl->r_slots, &pl->r_out), "resident");
        });
        st.kernel_launches += 1;
        st.forward_passes = 1;
        st.backward_passes = forward_only ? 0 : 1;
        st.observable_passes = forward_only ? 0 : 1;
        bytes = rb;
        st.passes_per_layer = 1;
        st.resident = 1;
    } else {
        const size_t NPS = P.steps.size();
        const bool ms = pl->memsave();
        const float2 *final_state = !NPS ? pl->psi0_src
                                    : ms  ? pl->W
                                          : pl->slots + size_t(P.n_slots - 1) * pl->amps_padded;
        auto slot16 = [&](size_t pi) { return pl->slots16 + P.slot_index(pi) * pl->amps_padded; };
        // layout A's tiles are contiguous runs of 4096 amplitudes (local qubits 0..11)
        const bool L0_contiguous = !P.layouts.empty() && P.layouts[0].tile_lo_bits == 0 &&
                                   P.layouts[0].row_start == 4;
        // forward (MemSave: every pass in place on W; a slot pass is narrowed into its bf16 slot)
        std::unique_ptr<Nvtx> range(new Nvtx("qfuse forward"));
        for (size_t pi = 0; pi < NPS; ++pi) {
            const PassStep &ps = P.steps[pi];
            const CUtensorMap *in;
            if (pi == 0) in = &pl->m_psi0[ps.layout];
            else if (!ms && P.slot_pass(pi - 1)) in = &pl->m_slot[P.slot_index(pi - 1)][ps.layout];
            else in = &pl->m_W[ps.layout];
            const CUtensorMap *outm = (!ms && P.slot_pass(pi)) ? &pl->m_slot[P.slot_index(pi)][ps.layout]
                                                               : &pl->m_W[ps.layout];
            PassParams p = pass_params(pl, ps, true);
            const bool wide = pass_is_wide(false, p);
            const bool narrow = ms && P.slot_pass(pi) && pi + 1 < NPS && !forward_only;
            if (narrow && wide && ps.layout == 0 && L0_contiguous) p.slot16 = slot16(pi); // fused narrow
            const int grid = wide ? std::min(wide_grid(pl->ctx->sms), p.tiles) : std::min(pl->grid_fwd, p.tiles);
            pl->timed(0, (p.slot16 ? 2.5 : 2.0) * sb, [&] { ck(launch_pass(s, false, grid, p, in, outm, nullptr), "pass fwd"); });
            st.kernel_launches++;
            st.forward_passes++;
            bytes += (p.slot16 ? 2.5 : 2.0) * sb;
            if (narrow && !p.slot16) {
                pl->timed(6, 1.5 * sb, [&] { ck(launch_narrow_bf16(s, pl->W, slot16(pi), pl->amps_padded), "narrow"); });
                st.kernel_launches++;
                bytes += 1.5 * sb;
            }
        }
        SeedParams sp{};
        sp.n = int(n);
        sp.batch = P.batch;
        sp.x_mask = P.x_mask;
        sp.z_mask = P.z_mask;
        sp.y_count = P.y_count;
        sp.wfinal = pl->wfinal;
        sp.czfinal = pl->final_adj;
        sp.psi = final_state;
        sp.lam = pl->lam;
        sp.epart = pl->epart;
        sp.apply_only = forward_only ? 1 : 0;
        range.reset(); // pop before the next push (NVTX ranges are a stack)
        range.reset(new Nvtx("qfuse observable"));
        pl->timed(2, 2 * sb, [&] { ck(launch_seed(s, sp), "seed"); });
        st.kernel_launches++;
        st.observable_passes++;
        bytes += 2 * sb;
        range.reset();
        range.reset(new Nvtx("qfuse backward"));
        if (!forward_only) {
            for (size_t pi = NPS; pi-- > 0;) {
                const PassStep &ps = P.bstep(pi);
                const bool from_slot = P.slot_pass(pi);
                const CUtensorMap *in = (from_slot && !ms) ? &pl->m_slot[P.slot_index(pi)][ps.layout]
                                                           : &pl->m_W[ps.layout];
                if (ms && from_slot && pi + 1 < NPS) { // re-anchor from the bf16 slot
                    // (W is free: the pass after a slot pass did not write psi)
                    pl->timed(6, 1.5 * sb, [&] { ck(launch_widen_bf16(s, slot16(pi), pl->W, pl->amps_padded), "widen"); });
                    st.kernel_launches++;
                    bytes += 1.5 * sb;
                }
                const bool write_psi = pi > 0 && !P.slot_pass(pi - 1);
                PassParams p = pass_params(pl, ps, write_psi, P.alt);
                pl->timed(1, (write_psi ? 4 : 3) * sb, [&] {
                    ck(launch_pass(s, true, pl->grid_bwd, p, in, &pl->m_W[ps.layout], &pl->m_lam[ps.layout]),
                       "pass bwd");
                });
                st.kernel_launches++;
                st.backward_passes++;
                bytes += (write_psi ? 4 : 3) * sb;
            }
        }
        range.reset();
        st.passes_per_layer = S ? uint32_t((NPS + S - 1) / S) : 0;
        st.resident = 0;
    }
    if (!forward_only) {
        const uint64_t chunks = (1ull << n) >= uint64_t(kTileAmps) ? (1ull << n) / kTileAmps : 1;
        const int grid_k = P.resident ? pl->grid_res : pl->grid_bwd;
        pl->timed(4, 0, [&] {
            ck(launch_reduce(s, (long long)S * n * 8, grid_k, pl->kpart, pl->kout,
                             P.resident ? nullptr : pl->epart, int(chunks), P.batch,
                             out_dev + P.n_params + 1),
               "reduce");
            ck(launch_zchain(s, int(S), int(n), pl->ry, pl->kout), "zchain");
            ck(launch_finalize(s, int(P.sec_q.size()), pl->sec_q, pl->sec_stage, pl->sec_off,
                               pl->sec_gates, pl->sec_gamma, theta_dev, int(n), pl->kout, out_dev,
                               out_dev + P.n_params + 1, P.batch, out_dev + P.n_params),
               "finalize");
        });
        st.kernel_launches += 3;
    }
    st.hbm_bytes = uint64_t(bytes);
    st.ckpt_layers = P.ckpt_layers;
    st.stages = S;
}

void enqueue_pergate(qf_plan *pl, const double *theta_dev, double *out_dev, qf_stats &st) {
    const Plan &P = pl->P;
    cudaStream_t s = pl->ctx->stream;
    const uint32_t n = P.n;
    const double sb = double(pl->amps) * 8.0;
    double bytes = 0;
    float2 *psi = P.resident ? pl->slots : pl->W;
    ck(cudaMemcpyAsync(psi, pl->psi0_src, pl->amps * 8, cudaMemcpyDeviceToDevice, s), "copy");
    for (const qf_gate &g : P.gates) {
        pl->timed(5, 2 * sb, [&] {
            ck(launch_gate_fwd(s, psi, int(n), P.batch, g.kind, g.axis, g.q0, g.q1, theta_dev, g.param), "gate fwd");
        });
        st.kernel_launches++;
        st.forward_passes++;
        bytes += 2 * sb;
    }
    ck(cudaMemsetAsync(pl->wfinal, 0, (n + 1) * sizeof(double), s), "memset");
    SeedParams sp{};
    sp.n = int(n);
    sp.batch = P.batch;
    sp.x_mask = P.x_mask;
    sp.z_mask = P.z_mask;
    sp.y_count = P.y_count;
    sp.wfinal = pl->wfinal;
    sp.czfinal = nullptr;
    sp.apply_only = 0;
    sp.psi = psi;
    sp.lam = pl->lam;
    sp.epart = pl->epart;
    ck(launch_seed(s, sp), "seed");
    st.kernel_launches++;
    st.observable_passes++;
    bytes += 2 * sb;
    int r = pl->n_rot;
    for (size_t i = P.gates.size(); i-- > 0;) {
        const qf_gate &g = P.gates[i];
        double *gp = nullptr;
        if (g.kind == QF_GATE_ROTATION) gp = pl->gpart + size_t(--r) * pl->gblocks;
        pl->timed(5, 4 * sb, [&] {
            ck(launch_gate_bwd(s, psi, pl->lam, int(n), P.batch, g.kind, g.axis, g.q0, g.q1,
                               theta_dev, g.param, gp),
               "gate bwd");
        });
        st.kernel_launches++;
        st.backward_passes++;
        bytes += 4 * sb;
    }
    ck(launch_gate_grad_reduce(s, pl->gpart, pl->gblocks, pl->rot_params, pl->n_rot, out_dev), "grad reduce");
    const uint64_t chunks = (1ull << n) >= uint64_t(kTileAmps) ? (1ull << n) / kTileAmps : 1;
    ck(launch_reduce(s, 0, 1, nullptr, nullptr, pl->epart, int(chunks), P.batch,
                     out_dev + P.n_params + 1),
       "reduce");
    ck(launch_finalize(s, 0, nullptr, nullptr, nullptr, nullptr, nullptr, theta_dev, int(n), nullptr,
                       out_dev, out_dev + P.n_params + 1, P.batch, out_dev + P.n_params),
       "finalize");
    st.kernel_launches += 3;
    st.hbm_bytes = uint64_t(bytes);
    st.passes_per_layer = P.layers ? uint32_t(P.gates.size() / P.layers) : 0;
}

void drop_cache(qf_ctx *ctx) {
    delete ctx->cached;
    ctx->cached = nullptr;
    ctx->cache_key.clear();
}

qf_plan *create_plan(qf_ctx *ctx, const qf_gate *gates, size_t n_gates, uint32_t n, uint32_t n_params,
                     uint32_t layers, uint32_t ckpt, uint32_t batch, uint64_t x, uint64_t z,
                     uint32_t storage = QF_STORAGE_FULL) {
    if (!ctx) throw std::invalid_argument("null context");
    if (storage != QF_STORAGE_FULL && storage != QF_STORAGE_MEMSAVE)
        throw std::invalid_argument("unknown storage mode");
    auto pl = std::make_unique<qf_plan>();
    pl->ctx = ctx;
    pl->storage = storage;
    pl->P = make_plan(gates, n_gates, n, n_params, layers, ckpt, batch, x, z);
    drop_cache(ctx); // the one-shot cache must not hold HBM a new plan needs
    build_device_plan(pl.get());
    return pl.release();
}

// Plan of a one-shot call: the context's cached plan when the call has the same
// gates, shape and storage mode as the last one, else a new plan (which then
// replaces the cache). `owned` is set when the caller must free it (cache off).
qf_plan *oneshot_plan(qf_ctx *ctx, const qf_gate *gates, size_t n_gates, uint32_t n, uint32_t n_params,
                      uint32_t layers, uint32_t ckpt, uint32_t batch, uint64_t x, uint64_t z,
                      uint32_t storage, bool &owned) {
    if (!ctx) throw std::invalid_argument("null context");
    if (n_gates && !gates) throw std::invalid_argument("null gate list");
    std::string key(sizeof(uint32_t) * 6 + sizeof(uint64_t) * 2 + n_gates * sizeof(qf_gate), '\0');
    char *k = key.data();
    const uint32_t head[6] = {n, n_params, layers, ckpt, batch, storage};
    const uint64_t masks[2] = {x, z};
    std::memcpy(k, head, sizeof(head));
    std::memcpy(k + sizeof(head), masks, sizeof(masks));
    if (n_gates) std::memcpy(k + sizeof(head) + sizeof(masks), gates, n_gates * sizeof(qf_gate));
    owned = false;
    if (ctx->cache_enabled && ctx->cached && ctx->cache_key == key) return ctx->cached;
    qf_plan *pl = create_plan(ctx, gates, n_gates, n, n_params, layers, ckpt, batch, x, z, storage);
    if (ctx->cache_enabled) {
        ctx->cached = pl;
        ctx->cache_key = std::move(key);
    } else {
        owned = true;
    }
    return pl;
}

// Host psi0 (pageable, the caller's BatchedState storage) -> the plan's psi0 through
// the context's pinned staging buffer: host threads copy 16 MiB chunks while the
// chunks already staged are DMA'd in order (copy and transfer overlap). Pinned
// sources and small states go straight to cudaMemcpyAsync.
void stage_psi0(qf_plan *pl, const float *src) {
    qf_ctx *c = pl->ctx;
    const size_t bytes = size_t(pl->amps) * 8;
    bind_psi0(pl, pl->psi0);
    cudaPointerAttributes attr{};
    const bool pinned = cudaPointerGetAttributes(&attr, src) == cudaSuccess && attr.type == cudaMemoryTypeHost;
    cudaGetLastError();
    if (pinned || bytes < (size_t(8) << 20)) {
        ck(cudaMemcpyAsync(pl->psi0, src, bytes, cudaMemcpyHostToDevice, c->stream), "H2D psi0");
        return;
    }
    ck(cudaStreamSynchronize(c->stream), "staging"); // no DMA still reads the staging buffer
    if (c->stage_bytes < bytes) {
        if (c->stage) cudaFreeHost(c->stage);
        c->stage = nullptr;
        c->stage_bytes = 0;
        void *h = nullptr;
        if (cudaMallocHost(&h, bytes) != cudaSuccess) {
            cudaGetLastError();
            throw CapacityError("pinned staging buffer of " + std::to_string(bytes >> 20) + " MiB failed");
        }
        c->stage = static_cast<float *>(h);
        c->stage_bytes = bytes;
    }
    constexpr size_t kChunk = size_t(16) << 20;
    const size_t nchunks = (bytes + kChunk - 1) / kChunk;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t T = std::min<size_t>({size_t(8), size_t(hw), nchunks});
    std::unique_ptr<std::atomic<int>[]> ready(new std::atomic<int>[nchunks]);
    for (size_t i = 0; i < nchunks; ++i) ready[i].store(0, std::memory_order_relaxed);
    char *dst = reinterpret_cast<char *>(c->stage);
    const char *from = reinterpret_cast<const char *>(src);
    auto work = [&](size_t t) {
        for (size_t i = t; i < nchunks; i += T) {
            const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
            std::memcpy(dst + off, from + off, len);
            ready[i].store(1, std::memory_order_release);
        }
    };
    struct Joiner {
        std::vector<std::thread> v;
        ~Joiner() {
            for (auto &t : v)
                if (t.joinable()) t.join();
        }
    } threads;
    for (size_t t = 0; t < T; ++t) threads.v.emplace_back(work, t);
    char *ddst = reinterpret_cast<char *>(pl->psi0);
    for (size_t i = 0; i < nchunks; ++i) {
        while (!ready[i].load(std::memory_order_acquire)) std::this_thread::yield();
        const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
        ck(cudaMemcpyAsync(ddst + off, dst + off, len, cudaMemcpyHostToDevice, c->stream), "H2D psi0");
    }
}

enum class Mode { Fused, PerGate };

void run_host(qf_plan *pl, const double *theta, double *loss, double *grad, double *expect,
              qf_stats *stats, Mode mode) {
    const Plan &P = pl->P;
    if (P.n_params && !theta) throw std::invalid_argument("gradient: theta length mismatch");
    if (!loss || (P.n_params && !grad)) throw std::invalid_argument("gradient: null output");
    ck(cudaSetDevice(pl->ctx->device), "cudaSetDevice");
    cudaStream_t s = pl->ctx->stream;
    qf_stats st{};
    if (P.n_params) std::memcpy(pl->h_theta, theta, sizeof(double) * P.n_params);
    ck(cudaEventRecord(pl->ev0, s), "event");
    if (P.n_params)
        ck(cudaMemcpyAsync(pl->theta, pl->h_theta, sizeof(double) * P.n_params, cudaMemcpyHostToDevice, s), "H2D");
    if (mode == Mode::Fused) {
        enqueue_fused(pl, pl->theta, pl->out, st);
    } else {
        if (!pl->gpart) pl->gpart = dalloc<double>(size_t(std::max(1, pl->n_rot)) * pl->gblocks, pl->owned);
        enqueue_pergate(pl, pl->theta, pl->out, st);
    }
    ck(cudaMemcpyAsync(pl->h_out, pl->out, sizeof(double) * pl->out_len(), cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaEventRecord(pl->ev1, s), "event");
    ck(cudaStreamSynchronize(s), "gradient");
    float ms = 0;
    cudaEventElapsedTime(&ms, pl->ev0, pl->ev1);
    st.device_ms = ms;
    st.device_bytes = pl->device_bytes;
    *loss = pl->h_out[P.n_params];
    if (P.n_params) std::memcpy(grad, pl->h_out, sizeof(double) * P.n_params);
    if (expect) std::memcpy(expect, pl->h_out + P.n_params + 1, sizeof(double) * P.batch);
    pl->last = st;
    if (stats) *stats = st;
}

// complex128 driver. fused: one HBM pass per segment (qf_c128_fused.cu);
// otherwise one per gate (qf_c128.cu, the reference's naive_gradient<double>).
// psi is uncomputed in place in fp64 either way (no checkpoint slots needed;
// ckpt_layers is validated like the complex64 path).
void run_c128(qf_ctx *ctx, const qf_gate *gates, size_t n_gates, uint32_t n_qubits,
              uint32_t n_params, uint32_t layers, uint32_t ckpt_layers, const double *psi0,
              uint32_t batch, const double *theta, uint64_t x_mask, uint64_t z_mask,
              double *loss_out, double *grad_out, double *expect_out, qf_stats *stats_out,
              bool fused) {
    if (!ctx) throw std::invalid_argument("null context");
    if (!psi0) throw std::invalid_argument("null psi0");
    // same validation (and error messages) as the complex64 path
    const Plan P = make_plan(gates, n_gates, n_qubits, n_params, layers, ckpt_layers, batch, x_mask, z_mask);
    if (P.n_params && !theta) throw std::invalid_argument("gradient: theta length mismatch");
    if (!loss_out || (P.n_params && !grad_out)) throw std::invalid_argument("gradient: null output");
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t s = ctx->stream;
    const uint32_t n = P.n;
    const uint64_t amps = uint64_t(batch) << n;
    const size_t state_bytes = size_t(amps) * sizeof(double2);
    const uint64_t dim = 1ull << n;
    const uint32_t chunks = dim >= 4096 ? uint32_t(dim / 4096) : 1u;
    std::vector<uint32_t> rp;
    for (const qf_gate &g : P.gates)
        if (g.kind == QF_GATE_ROTATION) rp.push_back(g.param);
    const int n_rot = int(rp.size());
    const C128Plan F = fused ? build_c128_plan(P.gates.data(), P.gates.size(), n, batch, ctx->sms) : C128Plan{};
    const int nsec = int(F.sec_off.size());
    const int seg_grid = fused ? c128_seg_grid(ctx->sms, uint64_t(batch) << (n - F.segs[0].m)) : 0;
    const int gblocks = fused ? 0 : c128_gate_grid(std::max<uint64_t>(1, amps / 2));
    const size_t scratch = fused ? (size_t(nsec) * 8 + size_t(seg_grid) * kC128MaxSec * 8 +
                                    size_t(nsec) * 8) * 8
                                 : size_t(std::max(1, n_rot)) * gblocks * 8;
    size_t free_b = 0, total_b = 0;
    ck(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
    const uint64_t budget = ctx->hbm_limit ? std::min<uint64_t>(ctx->hbm_limit, free_b) : free_b;
    const size_t need = 2 * state_bytes + scratch + (size_t(64) << 20);
    if (need > budget)
        throw CapacityError("device working set of " + std::to_string(need >> 20) +
                            " MiB exceeds the HBM budget of " + std::to_string(budget >> 20) + " MiB");
    std::vector<void *> owned;
    struct Free {
        std::vector<void *> &v;
        ~Free() {
            for (void *p : v) cudaFree(p);
        }
    } guard{owned};
    double2 *psi = dalloc<double2>(amps, owned), *lam = dalloc<double2>(amps, owned);
    double *th = dalloc<double>(std::max<uint32_t>(1, P.n_params), owned);
    double *epart = dalloc<double>(size_t(batch) * chunks, owned);
    double *out = dalloc<double>(size_t(P.n_params) + 1 + batch, owned);
    ck(cudaMemcpyAsync(psi, psi0, state_bytes, cudaMemcpyHostToDevice, s), "H2D psi0");
    if (P.n_params)
        ck(cudaMemcpyAsync(th, theta, sizeof(double) * P.n_params, cudaMemcpyHostToDevice, s), "H2D theta");
    ck(cudaMemsetAsync(out, 0, sizeof(double) * (size_t(P.n_params) + 1 + batch), s), "memset");
    double *grad_d = out, *loss_d = out + P.n_params, *exp_d = out + P.n_params + 1;
    qf_stats st{};
    struct Events {
        cudaEvent_t a = nullptr, b = nullptr;
        ~Events() {
            if (a) cudaEventDestroy(a);
            if (b) cudaEventDestroy(b);
        }
    } ev;
    ck(cudaEventCreate(&ev.a), "event");
    ck(cudaEventCreate(&ev.b), "event");
    ck(cudaEventRecord(ev.a, s), "event"); // device time: kernels only (psi0 already resident)
    if (fused) {
        C128Op *ops = dupload(F.ops, owned);
        C128Round *rounds = dupload(F.rounds, owned);
        uint32_t *cz = dupload(F.cz, owned);
        uint32_t *soff = dupload(F.sec_off, owned), *scnt = dupload(F.sec_cnt, owned),
                 *sgat = dupload(F.sec_gates, owned);
        double2 *secU = dalloc<double2>(size_t(std::max(1, nsec)) * kC128SecWords, owned);
        double *K = dalloc<double>(size_t(std::max(1, nsec)) * 8, owned);
        double *kpart = dalloc<double>(size_t(seg_grid) * kC128MaxSec * 8, owned);
        unsigned *ticket = dalloc<unsigned>(1, owned);
        ck(cudaMemsetAsync(ticket, 0, sizeof(unsigned), s), "memset");
        ck(launch_c128_prep(s, nsec, soff, scnt, sgat, th, secU), "c128 prep");
        for (const C128Seg &sg : F.segs) {
            ck(launch_c128_segment(s, false, seg_grid, sg, ops, rounds, cz, secU, psi, lam, int(n), batch,
                                   kpart, ticket, K),
               "c128 segment");
            st.forward_passes++;
        }
        ck(launch_seed_c128(s, int(n), batch, P.x_mask, P.z_mask, P.y_count, psi, lam, chunks, epart),
           "c128 seed");
        for (size_t i = F.segs.size(); i-- > 0;) {
            ck(launch_c128_segment(s, true, seg_grid, F.segs[i], ops, rounds, cz, secU, psi, lam, int(n),
                                   batch, kpart, ticket, K),
               "c128 segment");
            st.backward_passes++;
        }
        ck(launch_c128_finalize(s, nsec, soff, scnt, sgat, th, secU, K, grad_d), "c128 finalize");
        ck(launch_reduce_c128(s, nullptr, 0, nullptr, 0, grad_d, epart, chunks, batch, exp_d, loss_d),
           "c128 reduce");
        st.kernel_launches = st.forward_passes + st.backward_passes + 4;
    } else {
        double *gpart = dalloc<double>(size_t(std::max(1, n_rot)) * gblocks, owned);
        uint32_t *params = dupload(rp, owned);
        for (const qf_gate &g : P.gates) {
            ck(launch_gate_fwd_c128(s, psi, int(n), batch, g.kind, g.axis, g.q0, g.q1, th, g.param), "c128 fwd");
            st.forward_passes++;
        }
        ck(launch_seed_c128(s, int(n), batch, P.x_mask, P.z_mask, P.y_count, psi, lam, chunks, epart), "c128 seed");
        int r = n_rot;
        for (size_t i = P.gates.size(); i-- > 0;) {
            const qf_gate &g = P.gates[i];
            double *gp = g.kind == QF_GATE_ROTATION ? gpart + size_t(--r) * gblocks : nullptr;
            ck(launch_gate_bwd_c128(s, psi, lam, int(n), batch, g.kind, g.axis, g.q0, g.q1, th, g.param, gp),
               "c128 bwd");
            st.backward_passes++;
        }
        ck(launch_reduce_c128(s, gpart, gblocks, params, n_rot, grad_d, epart, chunks, batch, exp_d, loss_d),
           "c128 reduce");
        st.kernel_launches = st.forward_passes + st.backward_passes + 2;
    }
    ck(cudaEventRecord(ev.b, s), "event");
    std::vector<double> h(size_t(P.n_params) + 1 + batch);
    ck(cudaMemcpyAsync(h.data(), out, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "c128 gradient");
    float dev_ms = 0.f;
    ck(cudaEventElapsedTime(&dev_ms, ev.a, ev.b), "elapsed");
    st.device_ms = dev_ms;
    *loss_out = h[P.n_params];
    if (P.n_params) std::memcpy(grad_out, h.data(), sizeof(double) * P.n_params);
    if (expect_out) std::memcpy(expect_out, h.data() + P.n_params + 1, sizeof(double) * batch);
    st.observable_passes = 1;
    st.hbm_bytes = uint64_t((2.0 * st.forward_passes + 4.0 * st.backward_passes + 2.0) * state_bytes);
    st.device_bytes = 2 * state_bytes;
    st.passes_per_layer = P.layers ? uint32_t((st.forward_passes + P.layers - 1) / P.layers) : 0;
    st.stages = P.stages;
    if (stats_out) *stats_out = st;
}

} // namespace

extern "C" {

const char *qf_last_error(void) { return g_err.c_str(); }
const char *qf_version(void) { return "qfuse-b200 0.1.0 (sm_100a)"; }

int qf_ctx_create(int device, qf_ctx **out) {
    return guarded([&] {
        if (!out) throw std::invalid_argument("null output pointer");
        int count = 0;
        ck(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
        if (device < 0 || device >= count) throw std::invalid_argument("no such CUDA device");
        ck(cudaSetDevice(device), "cudaSetDevice");
        cudaDeviceProp prop;
        ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
        if (prop.major != 10)
            throw DeviceError("qfuse-b200 is built for sm_100a (Blackwell B200); device " +
                              std::string(prop.name) + " is sm_" + std::to_string(prop.major) +
                              std::to_string(prop.minor));
        auto c = std::make_unique<qf_ctx>();
        c->device = device;
        c->sms = prop.multiProcessorCount;
        ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
        *out = c.release();
    });
}

int qf_ctx_destroy(qf_ctx *ctx) {
    return guarded([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        drop_cache(ctx);
        if (ctx->stage) cudaFreeHost(ctx->stage);
        if (ctx->stream) cudaStreamDestroy(ctx->stream);
        delete ctx;
    });
}

int qf_ctx_set_hbm_limit(qf_ctx *ctx, uint64_t bytes) {
    return guarded([&] {
        if (!ctx) throw std::invalid_argument("null context");
        ctx->hbm_limit = bytes;
    });
}

int qf_ctx_set_plan_cache(qf_ctx *ctx, int enable) {
    return guarded([&] {
        if (!ctx) throw std::invalid_argument("null context");
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        ctx->cache_enabled = enable != 0;
        if (!enable) {
            drop_cache(ctx);
            if (ctx->stage) cudaFreeHost(ctx->stage);
            ctx->stage = nullptr;
            ctx->stage_bytes = 0;
        }
    });
}

int qf_plan_create(qf_ctx *ctx, const qf_gate *gates, size_t n_gates, uint32_t n_qubits,
                   uint32_t n_params, uint32_t layers, uint32_t ckpt_layers, uint32_t batch,
                   uint64_t x_mask, uint64_t z_mask, qf_plan **out) {
    return guarded([&] {
        if (!out) throw std::invalid_argument("null output pointer");
        *out = create_plan(ctx, gates, n_gates, n_qubits, n_params, layers, ckpt_layers, batch,
                           x_mask, z_mask);
    });
}

int qf_plan_create_ex(qf_ctx *ctx, const qf_gate *gates, size_t n_gates, uint32_t n_qubits,
                      uint32_t n_params, uint32_t layers, uint32_t ckpt_layers, uint32_t batch,
                      uint64_t x_mask, uint64_t z_mask, uint32_t storage_mode, qf_plan **out) {
    return guarded([&] {
        if (!out) throw std::invalid_argument("null output pointer");
        *out = create_plan(ctx, gates, n_gates, n_qubits, n_params, layers, ckpt_layers, batch,
                           x_mask, z_mask, storage_mode);
    });
}

int qf_plan_describe(const qf_gate *gates, size_t n_gates, uint32_t n_qubits, uint32_t n_params,
                     uint32_t layers, uint32_t ckpt_layers, uint32_t batch, uint64_t x_mask,
                     uint64_t z_mask, qf_plan_info *out) {
    return guarded([&] {
        if (!out) throw std::invalid_argument("null output pointer");
        const Plan P = make_plan(gates, n_gates, n_qubits, n_params, layers, ckpt_layers, batch,
                                 x_mask, z_mask);
        qf_plan_info info{};
        info.stages = P.stages;
        info.resident = P.resident ? 1u : 0u;
        info.slots = P.n_slots;
        const uint64_t S = uint64_t(8) << P.n; // bytes of one sample's state
        if (P.resident) {
            info.bytes_per_sample = S * (1 + 2 * uint64_t(P.n_slots));
        } else {
            const size_t NPS = P.steps.size();
            info.layouts = uint32_t(P.layouts.size());
            info.passes = uint32_t(NPS);
            info.ckpt_passes = P.ckpt_passes;
            info.balanced = P.alt ? 1u : 0u;
            auto prog_of = [&](const PassStep &ps) {
                const uint32_t rot = (ps.rot0 | ps.rot1) ? (ps.rot0 | ps.rot1) : P.layouts[ps.layout].rot_mask;
                return prog_encode(ps.nph, ps.ph, rot);
            };
            uint64_t units = 2; // observable: read psi, write lambda
            for (size_t pi = 0; pi < NPS; ++pi) {
                const PassStep &f = P.steps[pi];
                const uint32_t pf = prog_of(f);
                const bool wide = P.wide && f.layout == 0 && f.sd >= 0 && pf == kProgA;
                info.wide_forward += wide ? 1u : 0u;
                info.compiled_forward += (wide || prog_compiled(false, pf)) ? 1u : 0u;
                const PassStep &b = P.bstep(pi);
                const bool z = b.s0 == 0 || b.s1 == 0; // stage-0 Z measurement: runtime kernel
                info.compiled_backward += (!z && prog_compiled(true, prog_of(b))) ? 1u : 0u;
                units += 2 + ((pi > 0 && !P.slot_pass(pi - 1)) ? 4 : 3);
            }
            info.bytes_per_sample = S * units;
        }
        *out = info;
    });
}

int qf_plan_destroy(qf_plan *plan) {
    return guarded([&] { delete plan; });
}

int qf_plan_upload_psi0(qf_plan *plan, const float *psi0_host) {
    return guarded([&] {
        if (!plan || !psi0_host) throw std::invalid_argument("null argument");
        ck(cudaSetDevice(plan->ctx->device), "cudaSetDevice");
        bind_psi0(plan, plan->psi0);
        ck(cudaMemcpyAsync(plan->psi0, psi0_host, plan->amps * 8, cudaMemcpyHostToDevice,
                           plan->ctx->stream),
           "H2D psi0");
    });
}

int qf_plan_set_psi0_device(qf_plan *plan, const float *psi0_device) {
    return guarded([&] {
        if (!plan || !psi0_device) throw std::invalid_argument("null argument");
        ck(cudaSetDevice(plan->ctx->device), "cudaSetDevice");
        bind_psi0(plan, reinterpret_cast<const float2 *>(psi0_device)); // aliased, not copied
    });
}

int qf_plan_gradient(qf_plan *plan, const double *theta, double *loss_out, double *grad_out,
                     double *expect_out, qf_stats *stats_out) {
    return guarded([&] {
        if (!plan) throw std::invalid_argument("null plan");
        run_host(plan, theta, loss_out, grad_out, expect_out, stats_out, Mode::Fused);
    });
}

int qf_plan_gradient_pergate(qf_plan *plan, const double *theta, double *loss_out,
                             double *grad_out, double *expect_out, qf_stats *stats_out) {
    return guarded([&] {
        if (!plan) throw std::invalid_argument("null plan");
        run_host(plan, theta, loss_out, grad_out, expect_out, stats_out, Mode::PerGate);
    });
}

int qf_plan_gradient_device(qf_plan *plan, const double *theta_dev, double *out_dev) {
    return guarded([&] {
        if (!plan || !out_dev || (plan->P.n_params && !theta_dev))
            throw std::invalid_argument("null argument");
        ck(cudaSetDevice(plan->ctx->device), "cudaSetDevice");
        qf_stats st{};
        enqueue_fused(plan, theta_dev, out_dev, st);
        st.device_bytes = plan->device_bytes;
        plan->last = st;
    });
}

namespace {
// Forward-only readout of `plan` with host theta: the final state before the
// observable (global phase restored), complex64 to host.
void forward_state(qf_plan *plan, const double *theta, float *psi_out_host) {
    ck(cudaSetDevice(plan->ctx->device), "cudaSetDevice");
    const Plan &P = plan->P;
    cudaStream_t s = plan->ctx->stream;
    if (P.n_params) {
        if (!theta) throw std::invalid_argument("forward: theta length mismatch");
        std::memcpy(plan->h_theta, theta, sizeof(double) * P.n_params);
        ck(cudaMemcpyAsync(plan->theta, plan->h_theta, sizeof(double) * P.n_params,
                           cudaMemcpyHostToDevice, s),
           "H2D");
    }
    qf_stats st{};
    enqueue_fused(plan, plan->theta, plan->out, st, /*forward_only=*/true);
    ck(cudaMemcpyAsync(psi_out_host, plan->lam, plan->amps * 8, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "forward");
    plan->last = st;
}
} // namespace

int qf_plan_forward_state(qf_plan *plan, const double *theta, float *psi_out_host) {
    return guarded([&] {
        if (!plan || !psi_out_host) throw std::invalid_argument("null argument");
        forward_state(plan, theta, psi_out_host);
    });
}

int qf_forward_c64(qf_ctx *ctx, const qf_gate *gates, size_t n_gates, uint32_t n_qubits,
                   uint32_t n_params, uint32_t layers, const float *psi0, uint32_t batch,
                   const double *theta, float *psi_out, qf_stats *stats_out) {
    return guarded([&] {
        if (!psi0 || !psi_out) throw std::invalid_argument("null argument");
        bool owned = false;
        qf_plan *pl = oneshot_plan(ctx, gates, n_gates, n_qubits, n_params, layers, 0, batch, 0, 0,
                                   QF_STORAGE_FULL, owned);
        std::unique_ptr<qf_plan> own(owned ? pl : nullptr);
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        stage_psi0(pl, psi0);
        forward_state(pl, theta, psi_out);
        if (stats_out) *stats_out = pl->last;
    });
}

void *qf_plan_stream(qf_plan *plan) { return plan ? plan->ctx->stream : nullptr; }

int qf_plan_synchronize(qf_plan *plan) {
    return guarded([&] {
        if (!plan) throw std::invalid_argument("null plan");
        ck(cudaStreamSynchronize(plan->ctx->stream), "synchronize");
    });
}

int qf_plan_traffic(const qf_plan *plan, uint64_t *total_bytes, uint64_t *pass_bytes,
                    uint64_t *passes_per_gradient) {
    return guarded([&] {
        if (!plan) throw std::invalid_argument("null plan");
        const qf_stats &s = plan->last;
        if (total_bytes) *total_bytes = s.hbm_bytes;
        if (pass_bytes) *pass_bytes = plan->amps * 8;
        if (passes_per_gradient) *passes_per_gradient = s.forward_passes + s.backward_passes;
    });
}

int qf_gradient_c64(qf_ctx *ctx, const qf_gate *gates, size_t n_gates, uint32_t n_qubits,
                    uint32_t n_params, uint32_t layers, uint32_t ckpt_layers, const float *psi0,
                    uint32_t batch, const double *theta, uint64_t x_mask, uint64_t z_mask,
                    double *loss_out, double *grad_out, double *expect_out, qf_stats *stats_out) {
    return guarded([&] {
        if (!psi0) throw std::invalid_argument("null psi0");
        bool owned = false;
        qf_plan *pl = oneshot_plan(ctx, gates, n_gates, n_qubits, n_params, layers, ckpt_layers, batch,
                                   x_mask, z_mask, QF_STORAGE_FULL, owned);
        std::unique_ptr<qf_plan> own(owned ? pl : nullptr);
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        stage_psi0(pl, psi0);
        run_host(pl, theta, loss_out, grad_out, expect_out, stats_out, Mode::Fused);
    });
}

int qf_gradient_c64_ex(qf_ctx *ctx, const qf_gate *gates, size_t n_gates, uint32_t n_qubits,
                       uint32_t n_params, uint32_t layers, uint32_t ckpt_layers,
                       uint32_t storage_mode, const float *psi0, uint32_t batch,
                       const double *theta, uint64_t x_mask, uint64_t z_mask, double *loss_out,
                       double *grad_out, double *expect_out, qf_stats *stats_out) {
    return guarded([&] {
        if (!psi0) throw std::invalid_argument("null psi0");
        bool owned = false;
        qf_plan *pl = oneshot_plan(ctx, gates, n_gates, n_qubits, n_params, layers, ckpt_layers, batch,
                                   x_mask, z_mask, storage_mode, owned);
        std::unique_ptr<qf_plan> own(owned ? pl : nullptr);
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        stage_psi0(pl, psi0);
        run_host(pl, theta, loss_out, grad_out, expect_out, stats_out, Mode::Fused);
    });
}

int qf_gradient_pergate_c64(qf_ctx *ctx, const qf_gate *gates, size_t n_gates, uint32_t n_qubits,
                            uint32_t n_params, uint32_t layers, uint32_t ckpt_layers,
                            const float *psi0, uint32_t batch, const double *theta,
                            uint64_t x_mask, uint64_t z_mask, double *loss_out, double *grad_out,
                            double *expect_out, qf_stats *stats_out) {
    return guarded([&] {
        if (!psi0) throw std::invalid_argument("null psi0");
        bool owned = false;
        qf_plan *pl = oneshot_plan(ctx, gates, n_gates, n_qubits, n_params, layers, ckpt_layers, batch,
                                   x_mask, z_mask, QF_STORAGE_FULL, owned);
        std::unique_ptr<qf_plan> own(owned ? pl : nullptr);
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        stage_psi0(pl, psi0);
        run_host(pl, theta, loss_out, grad_out, expect_out, stats_out, Mode::PerGate);
    });
}

int qf_gradient_c128(qf_ctx *ctx, const qf_gate *gates, size_t n_gates, uint32_t n_qubits,
                     uint32_t n_params, uint32_t layers, uint32_t ckpt_layers, const double *psi0,
                     uint32_t batch, const double *theta, uint64_t x_mask, uint64_t z_mask,
                     double *loss_out, double *grad_out, double *expect_out, qf_stats *stats_out) {
    return guarded([&] {
        run_c128(ctx, gates, n_gates, n_qubits, n_params, layers, ckpt_layers, psi0, batch, theta,
                 x_mask, z_mask, loss_out, grad_out, expect_out, stats_out, /*fused=*/true);
    });
}

int qf_gradient_pergate_c128(qf_ctx *ctx, const qf_gate *gates, size_t n_gates, uint32_t n_qubits,
                             uint32_t n_params, uint32_t layers, uint32_t ckpt_layers,
                             const double *psi0, uint32_t batch, const double *theta,
                             uint64_t x_mask, uint64_t z_mask, double *loss_out, double *grad_out,
                             double *expect_out, qf_stats *stats_out) {
    return guarded([&] {
        run_c128(ctx, gates, n_gates, n_qubits, n_params, layers, ckpt_layers, psi0, batch, theta,
                 x_mask, z_mask, loss_out, grad_out, expect_out, stats_out, /*fused=*/false);
    });
}

} // extern "C"

extern "C" {

int qf_plan_random_psi0(qf_plan *plan, uint64_t seed, uint64_t first_sample) {
    return guarded([&] {
        if (!plan) throw std::invalid_argument("null plan");
        ck(cudaSetDevice(plan->ctx->device), "cudaSetDevice");
        const uint64_t dim = 1ull << plan->P.n;
        const uint64_t chunks = dim >= 4096 ? dim / 4096 : 1;
        if (!plan->rand_scratch)
            plan->rand_scratch = dalloc<double>(size_t(plan->P.batch) * chunks, plan->owned);
        ck(launch_random_state(plan->ctx->stream, seed, first_sample, int(plan->P.n), plan->P.batch,
                               plan->rand_scratch, plan->psi0),
           "random psi0");
        ck(cudaStreamSynchronize(plan->ctx->stream), "random psi0");
    });
}

int qf_plan_set_profiling(qf_plan *plan, int enable) {
    return guarded([&] {
        if (!plan) throw std::invalid_argument("null plan");
        plan->profiling = enable != 0;
    });
}

int qf_plan_profile(qf_plan *plan, qf_profile *out, int reset) {
    return guarded([&] {
        if (!plan) throw std::invalid_argument("null plan");
        ck(cudaSetDevice(plan->ctx->device), "cudaSetDevice");
        plan->harvest();
        if (out) {
            for (int k = 0; k < 8; ++k) {
                out->launches[k] = plan->prof_launches[k];
                out->ms[k] = plan->prof_ms[k];
                out->bytes[k] = plan->prof_bytes[k];
            }
        }
        if (reset) {
            for (int k = 0; k < 8; ++k) {
                plan->prof_launches[k] = 0;
                plan->prof_ms[k] = 0;
                plan->prof_bytes[k] = 0;
            }
        }
    });
}

} // extern "C"

extern "C" int qf_plan_download_psi0(qf_plan *plan, float *psi0_host) {
    return guarded([&] {
        if (!plan || !psi0_host) throw std::invalid_argument("null argument");
        ck(cudaSetDevice(plan->ctx->device), "cudaSetDevice");
        ck(cudaMemcpyAsync(psi0_host, plan->psi0_src, plan->amps * 8, cudaMemcpyDeviceToHost,
                           plan->ctx->stream),
           "D2H psi0");
        ck(cudaStreamSynchronize(plan->ctx->stream), "D2H psi0");
    });
}

extern "C" int qf_plan_last_stats(const qf_plan *plan, qf_stats *out) {
    return guarded([&] {
        if (!plan || !out) throw std::invalid_argument("null argument");
        *out = plan->last;
    });
}

// Error channel for the other translation units of the library (qf_multi.cpp).
void qfb::set_last_error(const char *msg) { g_err = msg ? msg : ""; }
