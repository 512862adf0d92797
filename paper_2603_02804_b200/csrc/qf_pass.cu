// Streaming fused pass (n > 12): one HBM round trip of the batch store per
// pass. Persistent CTAs walk the tiles of the pass layout; each tile is
// loaded by TMA (SWIZZLE_128B) into shared memory, transformed by 1-5 group
// phases (registers + FFMA2), and stored back by TMA while the next tile's
// load is already in flight (double buffer, mbarrier completion).
//
// A pass applies  Ry_{s0}(X) -> D -> Ry_{s1}(X)  on its resident qubits X,
// so with two alternating layouts (qubits 0..11 / 0..3 + top 8) every stage
// costs ONE pass (the diagonal commutes with everything but the Ry's of its
// own stage boundary). Backward passes undo the same ops on psi and lambda
// and accumulate K = sum psi lambda^dag per (stage, qubit) in fp64.
#include <cstdlib>

#include "qf_device.cuh"

namespace qfb {
namespace {

using namespace dev;

constexpr size_t kAccBytes = size_t(8) * 2 * 12 * 8 * sizeof(double); // [warp][round][bit][8]

// Shared pass prologue: Ry tables (rys), group scales (mgs) and the diagonal's
// register table (treg_s). When the pass applies a diagonal and the product F
// of all its group scales is >= 2^-40, the scales are folded into the
// diagonal (treg_s *= F) and the Ry rounds run unscaled: the tile is off by a
// known factor f between the diagonal and the round ends (|f| <= 2^40, no
// overflow), and the backward's K measurements, taken at f^2 x their true
// value, get kc = 1/f^2. Returns the scale flag for PhaseEnv.
__device__ bool pass_prologue(const PassParams &p, uint32_t tid, float4 *rys, float2 *treg_s,
                              float2 *mgs, float *kc) {
    if (tid < 24) {
        const int r = tid / 12, lb = tid % 12;
        const int s = r == 0 ? p.s0 : p.s1;
        float4 v = make_float4(0.f, 0.f, 1.f, 0.f); // identity: t = 0, m = 1
        if (s >= 0 && (((r == 0 ? p.rot0 : p.rot1) >> lb) & 1u)) v = ry_entry(p.ry[size_t(s) * p.n + p.qmap[lb]]);
        rys[tid] = v;
    } else if (tid >= 40 && tid < 46) { // product of the factored m per (round, group)
        const int r = (tid - 40) / 3, g = (tid - 40) % 3;
        const int s = r == 0 ? p.s0 : p.s1;
        float M = 1.f;
        for (int b = 0; b < 4; ++b) {
            const int lb = 4 * g + b;
            if (s >= 0 && (((r == 0 ? p.rot0 : p.rot1) >> lb) & 1u)) M *= ry_entry(p.ry[size_t(s) * p.n + p.qmap[lb]]).z;
        }
        mgs[tid - 40] = make_float2(M, M);
    }
    __syncthreads();
    float F = 1.f;
#pragma unroll
    for (int i = 0; i < 6; ++i) F *= mgs[i].x;
    const bool fold = p.dt != nullptr && F >= 0x1p-40f;
    if (tid < 16) {
        float2 t = p.dt ? p.dt->treg[tid] : make_float2(1.f, 0.f);
        if (fold) t = make_float2(t.x * F, t.y * F);
        treg_s[tid] = t;
    } else if (tid == 16 && kc) { // backward order: phases nph-1 .. 0
        float f = 1.f;
        for (int i = 0; i < 6; ++i) kc[i] = 1.f;
        if (fold)
            for (int i = p.nph - 1; i >= 0; --i) {
                const int g = p.ph[i].g, ops = p.ph[i].ops;
                if (ops & 4) { f /= mgs[3 + g].x; kc[3 + g] = 1.f / (f * f); }
                if (ops & 2) f *= F;
                if (ops & 1) { f /= mgs[g].x; kc[g] = 1.f / (f * f); }
            }
    }
    __syncthreads();
    return !fold;
}

// Forward: 3 CTAs/SM, each double-buffered (load of tile i+1 overlaps tile i).
// Backward, NB = 1: 2 CTAs/SM, single-buffered (psi + lambda = 64 KiB); the two
// CTAs overlap each other's TMA traffic with compute. NB = 3: 1 CTA/SM with a
// 3-deep ring (load i+1 and store i-1 overlap tile i). Selected at plan time
// (QF_BWD_PIPE=3 for the ring).
constexpr size_t pass_smem(bool bwd, int nb) {
    return size_t(nb) * kTileBytes * (bwd ? 2 : 1) + 64 /*mbar*/ + 24 * 16 /*rys*/ +
           16 * 8 /*treg*/ + 8 * 8 /*mgs*/ + 32 /*kc*/ + (bwd ? kAccBytes : 0) + 1024 /*align*/;
}
constexpr int min_blocks(bool bwd, int nb) { return bwd ? (nb == 1 ? 2 : 1) : 3; }

template <bool BWD, int NB, uint32_t PROG = 0>
__global__ void __launch_bounds__(kThreads, min_blocks(BWD, NB))
    pass_kernel(const __grid_constant__ PassParams p, const __grid_constant__ CUtensorMap m_in,
                const __grid_constant__ CUtensorMap m_out,
                const __grid_constant__ CUtensorMap m_lam) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    constexpr uint32_t kBuf = uint32_t(kTileBytes) * (BWD ? 2 : 1);
    uint8_t *tail = smem + NB * kBuf;
    uint64_t *mbar = reinterpret_cast<uint64_t *>(tail);
    float4 *rys = reinterpret_cast<float4 *>(tail + 64);
    float2 *treg_s = reinterpret_cast<float2 *>(tail + 64 + 24 * 16);
    float2 *mgs = treg_s + 16; // [2 rounds][3 groups]
    float *kc = reinterpret_cast<float *>(tail + 64 + 24 * 16 + 16 * 8 + 8 * 8);
    double *acc = reinterpret_cast<double *>(tail + 64 + 24 * 16 + 16 * 8 + 8 * 8 + 32);
    const uint32_t tid = threadIdx.x, warp = tid >> 5;

    const int lo_mask = (1 << p.tile_lo_bits) - 1, hi_mask = (1 << p.tile_hi_bits) - 1;
    const int sample_shift = p.tile_lo_bits + p.tile_hi_bits;
    const uint32_t tis_mask = (1u << sample_shift) - 1u;
    auto issue_load = [&](int t, int b) {
        const int c1 = t & lo_mask, c3 = (t >> p.tile_lo_bits) & hi_mask, c4 = t >> sample_shift;
        uint8_t *dst = smem + b * kBuf;
        mbar_expect_tx(&mbar[b], kBuf);
        tma_load5(dst, &m_in, &mbar[b], 0, c1, 0, c3, c4);
        if (BWD) tma_load5(dst + kTileBytes, &m_lam, &mbar[b], 0, c1, 0, c3, c4);
    };
    const int stride = gridDim.x;
    if (tid == 0) { // first loads in flight before the prologue
        prefetch_map(&m_in);
        prefetch_map(&m_out);
        if (BWD) prefetch_map(&m_lam);
        for (int b = 0; b < NB; ++b) mbar_init(&mbar[b], 1);
        fence_mbar_init();
        for (int b = 0; b < NB; ++b)
            if (int(blockIdx.x) + b * stride < p.tiles) issue_load(blockIdx.x + b * stride, b);
    }
    if (BWD) {
        for (uint32_t i = tid; i < kAccBytes / 8; i += kThreads) acc[i] = 0.0;
    }
    const bool scale = pass_prologue(p, tid, rys, treg_s, mgs, BWD ? kc : nullptr);
    const float2 tthr = p.dt ? p.dt->tthr[tid] : make_float2(1.f, 0.f);
    const uint32_t thrinfo = p.cz ? p.cz->thrinfo[tid] : 0u;
    PhaseEnv env;
    env.rys = rys;
    env.mgs = mgs;
    env.rot = p.rot_mask;
    env.scale = scale;
    env.scale1 = scale;
    env.treg_s = treg_s;
    env.kc = BWD ? kc : nullptr;
    env.zm = uint32_t(p.zmask);
    env.acc_w = acc + warp * 2 * 12 * 8;
    env.acc_w1 = env.acc_w + 12 * 8;
    env.d.base = make_float2(1.f, 0.f);
    env.d.sgn = 0;
    int it = 0;
    for (int t = blockIdx.x; t < p.tiles; t += stride, ++it) {
        const int b = it % NB;
        if (p.dt) env.d = diag_ctx(tid, tthr, thrinfo, p.dt, p.cz, p.tileinfo, uint32_t(t) & tis_mask);
        mbar_wait(&mbar[b], (it / NB) & 1);
        uint8_t *pt = smem + b * kBuf;
        if (!BWD && PROG) {
            prog_fwd<PROG, 0>(pt, tid, env, [](auto cross) {
                if constexpr (decltype(cross)::value) __syncthreads();
                else __syncwarp();
            });
        } else if (!BWD) {
            for (int i = 0; i < p.nph; ++i) {
                if (i) __syncthreads();
                run_phase_fwd(p.ph[i].g, pt, tid, p.ph[i].ops, env);
            }
        } else {
            for (int i = p.nph - 1; i >= 0; --i) {
                if (i != p.nph - 1) __syncthreads();
                run_phase_bwd(p.ph[i].g, pt, pt + kTileBytes, tid, p.ph[i].ops, env);
            }
        }
        fence_async_smem();
        __syncthreads();
        if (tid == 0) {
            const int c1 = t & lo_mask, c3 = (t >> p.tile_lo_bits) & hi_mask, c4 = t >> sample_shift;
            if (!BWD || p.write_psi) tma_store5(&m_out, pt, 0, c1, 0, c3, c4);
            if (BWD) tma_store5(&m_lam, pt + kTileBytes, 0, c1, 0, c3, c4);
            bulk_commit();
            const int tn = t + NB * stride;
            if (tn < p.tiles) {
                bulk_wait_read0();
                issue_load(tn, b);
            }
        }
    }
    if (tid == 0) bulk_wait0();
    if (BWD) {
        __syncthreads();
        if (tid < 2 * 12 * 8) {
            const int r = tid / 96, lb = (tid / 8) % 12, c = tid & 7;
            const int s = r == 0 ? p.s0 : p.s1;
            if (s >= 0 && (((r == 0 ? p.rot0 : p.rot1) >> lb) & 1u)) {
                double sum = 0.0;
#pragma unroll
                for (int w = 0; w < 8; ++w) sum += acc[((w * 2 + r) * 12 + lb) * 8 + c];
                p.kpart[size_t(blockIdx.x) * size_t(p.kstride) + size_t(s) * p.n * 8 +
                        size_t(p.qmap[lb]) * 8 + c] = sum;
            }
        }
    }
}

// Backward, "dual": one 512-thread CTA per SM whose two 256-thread halves
// each process their own tile (named barriers 1, 2) over a shared ring of three
// psi+lambda buffers: 16 warps per SM like two CTAs, plus a prefetched tile.
// Tile k of the CTA (k = 0, 1, ...) is processed by half k % 2, lives in
// buffer k % 3 and completes mbarrier k % 6 (so no waiter can run two phases
// ahead of a barrier).
constexpr int kDualThreads = 2 * kThreads;
constexpr size_t kDualAcc = size_t(16) * 2 * 12 * 8 * sizeof(double);
constexpr size_t dual_smem() {
    return size_t(3) * 2 * kTileBytes + 64 /*6 mbar*/ + 24 * 16 + 16 * 8 + 8 * 8 + 32 + kDualAcc + 1024;
}
__device__ __forceinline__ void named_bar(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <uint32_t PROG = 0>
__global__ void __launch_bounds__(kDualThreads, 1)
    pass_bwd_dual(const __grid_constant__ PassParams p, const __grid_constant__ CUtensorMap m_in,
                  const __grid_constant__ CUtensorMap m_out,
                  const __grid_constant__ CUtensorMap m_lam) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    constexpr uint32_t kBuf = uint32_t(kTileBytes) * 2;
    uint8_t *tail = smem + 3 * kBuf;
    uint64_t *mbar = reinterpret_cast<uint64_t *>(tail);
    float4 *rys = reinterpret_cast<float4 *>(tail + 64);
    float2 *treg_s = reinterpret_cast<float2 *>(tail + 64 + 24 * 16);
    float2 *mgs = treg_s + 16;
    float *kc = reinterpret_cast<float *>(tail + 64 + 24 * 16 + 16 * 8 + 8 * 8);
    double *acc = reinterpret_cast<double *>(tail + 64 + 24 * 16 + 16 * 8 + 8 * 8 + 32);
    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    const int half = int(tid >> 8);
    const uint32_t gtid = tid & 255u;
    // light passes (layout B) are bound by the one-tile-deep ring: their next ring
    // load is prefetched into L2 (QF_L2PF=0 disables)
#ifndef QF_L2PF_NPH // (4-phase programs measured with the prefetch: +0.4% backward time)
#define QF_L2PF_NPH 3
#endif
    const bool L2PF = PROG != 0 && prog_nph(PROG) <= QF_L2PF_NPH && p.l2pf;

    const int lo_mask = (1 << p.tile_lo_bits) - 1, hi_mask = (1 << p.tile_hi_bits) - 1;
    const int sample_shift = p.tile_lo_bits + p.tile_hi_bits;
    const uint32_t tis_mask = (1u << sample_shift) - 1u;
    const int stride = gridDim.x;
    auto tile_of = [&](int k) { return int(blockIdx.x) + k * stride; };
    auto issue_load = [&](int k) {
        const int t = tile_of(k);
        const int c1 = t & lo_mask, c3 = (t >> p.tile_lo_bits) & hi_mask, c4 = t >> sample_shift;
        uint8_t *dst = smem + (k % 3) * kBuf;
        uint64_t *bar = &mbar[k % 6];
        mbar_expect_tx(bar, kBuf);
        tma_load5(dst, &m_in, bar, 0, c1, 0, c3, c4);
        tma_load5(dst + kTileBytes, &m_lam, bar, 0, c1, 0, c3, c4);
    };
    if (tid == 0) { // first loads in flight before the prologue
        prefetch_map(&m_in);
        prefetch_map(&m_out);
        prefetch_map(&m_lam);
        for (int b = 0; b < 6; ++b) mbar_init(&mbar[b], 1);
        fence_mbar_init();
        for (int k = 0; k < 3; ++k)
            if (tile_of(k) < p.tiles) issue_load(k);
    }
    for (uint32_t i = tid; i < kDualAcc / 8; i += kDualThreads) acc[i] = 0.0;
    const bool scale = pass_prologue(p, tid, rys, treg_s, mgs, kc);
    const float2 tthr = p.dt ? p.dt->tthr[gtid] : make_float2(1.f, 0.f);
    const uint32_t thrinfo = p.cz ? p.cz->thrinfo[gtid] : 0u;

    PhaseEnv env;
    env.rys = rys;
    env.mgs = mgs;
    env.rot = p.rot_mask;
    env.scale = scale;
    env.scale1 = scale;
    env.treg_s = treg_s;
    env.kc = kc;
    env.zm = uint32_t(p.zmask);
    env.acc_w = acc + warp * 2 * 12 * 8;
    env.acc_w1 = env.acc_w + 12 * 8;
    // Compiled programs accumulate (X, Y) per lane in fp32 registers (kmeasure
    // kslot) and move them into this warp's fp64 slots every 16 tiles and at the
    // end, so no fp32 sum runs over more than 16 tile partials.
    float kreg[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    env.kreg = kreg;
    auto kreg_flush = [&] {
        const uint32_t lane = tid & 31u;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            float r = kreg[i];
            r += __shfl_xor_sync(0xffffffffu, r, 8);
            r += __shfl_xor_sync(0xffffffffu, r, 16);
            const int rr = i / 3, g = i % 3, bit = int(lane >> 1), comp = int(lane & 1u);
            if (lane < 8 && (((rr == 0 ? p.rot0 : p.rot1) >> (4 * g + bit)) & 1u))
                acc[((warp * 2 + rr) * 12 + 4 * g + bit) * 8 + comp] += double(r);
            kreg[i] = 0.f;
        }
    };
    env.d.base = make_float2(1.f, 0.f);
    env.d.sgn = 0;
    const int bar_id = 1 + half;
    // The refill of a stored buffer (tile k + 3, for the other half) waits for
    // the store's shared-memory read; it is deferred to the end of this half's
    // next first phase, so no thread idles on the store.
    int pending = -1;
    for (int k = half; tile_of(k) < p.tiles; k += 2) {
        const int t = tile_of(k);
        if (p.dt) env.d = diag_ctx(gtid, tthr, thrinfo, p.dt, p.cz, p.tileinfo, uint32_t(t) & tis_mask);
        if (L2PF && gtid == 0 && tile_of(k + 3) < p.tiles) { // the next ring load, into L2 now
            const int tq = tile_of(k + 3);
            const int c1 = tq & lo_mask, c3 = (tq >> p.tile_lo_bits) & hi_mask, c4 = tq >> sample_shift;
            tma_prefetch5(&m_in, 0, c1, 0, c3, c4);
            tma_prefetch5(&m_lam, 0, c1, 0, c3, c4);
        }
        mbar_wait(&mbar[k % 6], (k / 6) & 1);
        uint8_t *pt = smem + (k % 3) * kBuf;
        auto refill = [&] {
            if (gtid == 0 && pending >= 0) {
                bulk_wait_read0();
                issue_load(pending);
                pending = -1;
            }
        };
#if QF_ABLATE_PHASES
        if (true) {
            refill();
        } else
#endif
        if constexpr (PROG != 0) {
            prog_bwd<PROG, int(prog_nph(PROG)) - 1>(pt, pt + kTileBytes, gtid, env, [&](auto cross) {
                refill();
                if constexpr (decltype(cross)::value) named_bar(bar_id, kThreads);
                else __syncwarp();
            });
            refill(); // single-phase programs
        } else {
            for (int i = p.nph - 1; i >= 0; --i) {
                if (i != p.nph - 1) named_bar(bar_id, kThreads);
                run_phase_bwd(p.ph[i].g, pt, pt + kTileBytes, gtid, p.ph[i].ops, env);
                if (i == p.nph - 1) refill();
            }
        }
        if constexpr (PROG != 0) {
            if (((k >> 1) & 15) == 15) kreg_flush(); // every 16 tiles of this half
        }
        fence_async_smem();
        named_bar(bar_id, kThreads);
        if (gtid == 0) {
            const int c1 = t & lo_mask, c3 = (t >> p.tile_lo_bits) & hi_mask, c4 = t >> sample_shift;
            if (p.write_psi) tma_store5(&m_out, pt, 0, c1, 0, c3, c4);
            tma_store5(&m_lam, pt + kTileBytes, 0, c1, 0, c3, c4);
            bulk_commit();
            if (tile_of(k + 3) < p.tiles) pending = k + 3;
        }
    }
    if (gtid == 0) {
        if (pending >= 0) { // unreachable: k + 3 exists only if k + 2 does
            bulk_wait_read0();
            issue_load(pending);
        }
        bulk_wait0();
    }
    if constexpr (PROG != 0) kreg_flush();
    __syncthreads();
    if (tid < 2 * 12 * 8) {
        const int r = tid / 96, lb = (tid / 8) % 12, c = tid & 7;
        const int s = r == 0 ? p.s0 : p.s1;
        if (s >= 0 && (((r == 0 ? p.rot0 : p.rot1) >> lb) & 1u)) {
            double sum = 0.0;
#pragma unroll
            for (int w = 0; w < 16; ++w) sum += acc[((w * 2 + r) * 12 + lb) * 8 + c];
            p.kpart[size_t(blockIdx.x) * size_t(p.kstride) + size_t(s) * p.n * 8 +
                    size_t(p.qmap[lb]) * 8 + c] = sum;
        }
    }
}

// Backward pipeline: 2 = dual (default; measured 9% faster than 1 on the
// 20q workload), 1 = two CTAs/SM single-buffered, 3 = 1 CTA/SM ring
// (QF_BWD_PIPE overrides, for A/B measurements).
int bwd_pipe() {
    static int nb = [] {
        const char *e = getenv("QF_BWD_PIPE");
        const int v = e ? atoi(e) : 2;
        return (v == 1 || v == 3) ? v : 2;
    }();
    return nb;
}

std::atomic<uint64_t> g_attrs{0};
template <class K> cudaError_t set_smem(K kernel, size_t bytes) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
}
cudaError_t ensure_attrs() {
    return once_per_device(g_attrs, [] {
        cudaError_t e = set_smem(pass_kernel<false, 2>, pass_smem(false, 2));
        if (e == cudaSuccess) e = set_smem(pass_kernel<false, 2, kProgA>, pass_smem(false, 2));
        if (e == cudaSuccess) e = set_smem(pass_kernel<false, 2, kProgB20>, pass_smem(false, 2));
        if (e == cudaSuccess) e = set_smem(pass_kernel<false, 2, kProgB16>, pass_smem(false, 2));
        if (e == cudaSuccess) e = set_smem(pass_kernel<false, 2, kProgB16x>, pass_smem(false, 2));
        if (e == cudaSuccess) e = set_smem(pass_kernel<true, 1>, pass_smem(true, 1));
        if (e == cudaSuccess) e = set_smem(pass_kernel<true, 3>, pass_smem(true, 3));
        if (e == cudaSuccess) e = set_smem(pass_bwd_dual<0>, dual_smem());
        if (e == cudaSuccess) e = set_smem(pass_bwd_dual<kProgA>, dual_smem());
        if (e == cudaSuccess) e = set_smem(pass_bwd_dual<kProgB20>, dual_smem());
        if (e == cudaSuccess) e = set_smem(pass_bwd_dual<kProgB16>, dual_smem());
        if (e == cudaSuccess) e = set_smem(pass_bwd_dual<kProgB16x>, dual_smem());
        if (e == cudaSuccess) e = set_smem(pass_bwd_dual<kProgAlt>, dual_smem());
        if (e == cudaSuccess) e = set_smem(pass_kernel<false, 2, kProgB20P>, pass_smem(false, 2));
        if (e == cudaSuccess) e = set_smem(pass_bwd_dual<kProgB20P>, dual_smem());
        if (e == cudaSuccess) e = set_smem(pass_bwd_dual<kProgAltP>, dual_smem());
        if (e == cudaSuccess) e = set_smem(pass_kernel<false, 2, kProgB16xP>, pass_smem(false, 2));
        if (e == cudaSuccess) e = set_smem(pass_bwd_dual<kProgB16xP>, dual_smem());
        return e;
    });
}

// QF_PROGS=0 forces the runtime-dispatch kernels (A/B timing).
bool progs_enabled() {
    static const bool v = [] {
        const char *e = getenv("QF_PROGS");
        return !e || atoi(e) != 0;
    }();
    return v;
}

} // namespace

size_t pass_smem_bytes(bool backward) {
    if (!backward) return pass_smem(false, 2);
    return bwd_pipe() == 2 ? dual_smem() : pass_smem(true, bwd_pipe());
}

int pass_occupancy(bool backward) {
    if (ensure_attrs() != cudaSuccess) return 0;
    int blocks = 0;
    if (!backward)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, pass_kernel<false, 2>, kThreads, pass_smem(false, 2));
    else if (bwd_pipe() == 3)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, pass_kernel<true, 3>, kThreads, pass_smem(true, 3));
    else if (bwd_pipe() == 2)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, pass_bwd_dual<0>, kDualThreads, dual_smem());
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, pass_kernel<true, 1>, kThreads, pass_smem(true, 1));
    return blocks;
}

bool prog_compiled(bool backward, uint32_t prog) {
    if (prog == 0 || !progs_enabled()) return false;
    if (prog == kProgA || prog == kProgB20 || prog == kProgB16 || prog == kProgB16x ||
        prog == kProgB20P || prog == kProgB16xP)
        return true;
    return backward && (prog == kProgAlt || prog == kProgAltP);
}

bool pass_is_wide(bool backward, const PassParams &p) {
    static const bool enabled = [] {
        const char *e = getenv("QF_WIDE"); // QF_WIDE=0: narrow kernels only (A/B timing)
        return !e || atoi(e) != 0;
    }();
    return enabled && !backward && p.dtw != nullptr && progs_enabled() && p.prog == kProgA;
}

cudaError_t launch_pass(cudaStream_t st, bool backward, int grid, const PassParams &p,
                        const CUtensorMap *psi_in, const CUtensorMap *psi_out,
                        const CUtensorMap *lam) {
    if (pass_is_wide(backward, p)) return launch_pass_wide(st, grid, p, psi_in, psi_out);
    cudaError_t e = ensure_attrs();
    if (e != cudaSuccess) return e;
    const CUtensorMap &l = lam ? *lam : *psi_out;
    // straight-line kernels for the compiled programs (Z is measured at stage 0 only:
    // those passes take the runtime-dispatch kernel)
    const uint32_t prog = progs_enabled() && !(backward && p.zmask) ? p.prog : 0u;
    if (!backward) {
        const size_t sm = pass_smem(false, 2);
        if (prog == kProgA) pass_kernel<false, 2, kProgA><<<grid, kThreads, sm, st>>>(p, *psi_in, *psi_out, l);
        else if (prog == kProgB20) pass_kernel<false, 2, kProgB20><<<grid, kThreads, sm, st>>>(p, *psi_in, *psi_out, l);
        else if (prog == kProgB16) pass_kernel<false, 2, kProgB16><<<grid, kThreads, sm, st>>>(p, *psi_in, *psi_out, l);
        else if (prog == kProgB16x) pass_kernel<false, 2, kProgB16x><<<grid, kThreads, sm, st>>>(p, *psi_in, *psi_out, l);
        else if (prog == kProgB20P) pass_kernel<false, 2, kProgB20P><<<grid, kThreads, sm, st>>>(p, *psi_in, *psi_out, l);
        else if (prog == kProgB16xP) pass_kernel<false, 2, kProgB16xP><<<grid, kThreads, sm, st>>>(p, *psi_in, *psi_out, l);
        else pass_kernel<false, 2><<<grid, kThreads, sm, st>>>(p, *psi_in, *psi_out, l);
    } else if (bwd_pipe() == 3) {
        pass_kernel<true, 3><<<grid, kThreads, pass_smem(true, 3), st>>>(p, *psi_in, *psi_out, l);
    } else if (bwd_pipe() == 2) {
        const size_t sm = dual_smem();
        if (prog == kProgA) pass_bwd_dual<kProgA><<<grid, kDualThreads, sm, st>>>(p, *psi_in, *psi_out, l);
        else if (prog == kProgB20) pass_bwd_dual<kProgB20><<<grid, kDualThreads, sm, st>>>(p, *psi_in, *psi_out, l);
        else if (prog == kProgB16) pass_bwd_dual<kProgB16><<<grid, kDualThreads, sm, st>>>(p, *psi_in, *psi_out, l);
        else if (prog == kProgB16x) pass_bwd_dual<kProgB16x><<<grid, kDualThreads, sm, st>>>(p, *psi_in, *psi_out, l);
        else if (prog == kProgAlt) pass_bwd_dual<kProgAlt><<<grid, kDualThreads, sm, st>>>(p, *psi_in, *psi_out, l);
        else if (prog == kProgB20P) pass_bwd_dual<kProgB20P><<<grid, kDualThreads, sm, st>>>(p, *psi_in, *psi_out, l);
        else if (prog == kProgAltP) pass_bwd_dual<kProgAltP><<<grid, kDualThreads, sm, st>>>(p, *psi_in, *psi_out, l);
        else if (prog == kProgB16xP) pass_bwd_dual<kProgB16xP><<<grid, kDualThreads, sm, st>>>(p, *psi_in, *psi_out, l);
        else pass_bwd_dual<0><<<grid, kDualThreads, sm, st>>>(p, *psi_in, *psi_out, l);
    } else {
        pass_kernel<true, 1><<<grid, kThreads, pass_smem(true, 1), st>>>(p, *psi_in, *psi_out, l);
    }
    return cudaGetLastError();
}

} // namespace qfb
