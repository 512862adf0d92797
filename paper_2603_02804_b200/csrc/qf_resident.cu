// Sample-resident kernel (n <= 12) and the observable step.
//
// n <= 12: one 4096-amplitude tile holds 2^(12-n) whole samples, so the
// forward over every stage, the observable (expectation + adjoint seed) and
// the adjoint backward run without leaving shared memory. HBM sees psi0 and
// the checkpoint slots (used to re-anchor the psi uncompute every k stages).
//
// Observable (engine.cpp:346-435): lambda = 2 O' psi, E_s = <psi|O'|psi>,
// with the circuit's final diagonal folded in, O' = D_f^dag O D_f.
// scalar complex products in the diagonal (packed FMUL2/FFMA2 measured -0.3% here)
#define QF_DIAG2 0
#include "qf_device.cuh"

namespace qfb {
namespace {

using namespace dev;

__device__ __forceinline__ uint32_t qform_adj(const CzAdj *cz, uint32_t v) {
    uint32_t par = 0, w = v;
    while (w) {
        const int q = __ffs(w) - 1;
        w &= w - 1;
        par ^= __popc(v & cz->adjlo[q]);
    }
    return par & 1u;
}

// 2 * phase_O(t) * D_f(t) * conj(D_f(x)), t = x ^ X (pauli_phase engine.cpp:346-372).
__device__ __forceinline__ float2 seed_factor(uint32_t x, uint64_t X, uint64_t Z, uint32_t y,
                                              const double *wf, const CzAdj *czf) {
    const uint32_t t = x ^ uint32_t(X);
    double ang = 0.0;
    uint32_t xm = uint32_t(X);
    while (xm) {
        const int q = __ffs(xm) - 1;
        xm &= xm - 1;
        ang += ((x >> q) & 1u) ? -wf[q] : wf[q];
    }
    uint32_t par = __popc(t & uint32_t(Z));
    if (czf) par += qform_adj(czf, x) ^ qform_adj(czf, t);
    double s, c;
    sincos(ang, &s, &c);
    double re = 2.0 * c, im = 2.0 * s;
    if (par & 1u) {
        re = -re;
        im = -im;
    }
    double r2 = re, i2 = im;
    switch (y & 3u) {
    case 1: r2 = -im; i2 = re; break;
    case 2: r2 = -re; i2 = -im; break;
    case 3: r2 = im; i2 = -re; break;
    default: break;
    }
    return make_float2(float(r2), float(i2));
}
// D_f(x) for the forward-state readout.
// wf[n]: the global phase (launch_phase_sum), so the readout equals the reference's
// forward<T> amplitude for amplitude (engine.hpp:131-133).
__device__ __forceinline__ float2 dfinal(uint32_t x, int n, const double *wf, const CzAdj *czf) {
    double ang = wf[n];
    for (int q = 0; q < n; ++q)
        if ((x >> q) & 1u) ang += wf[q];
    double s, c;
    sincos(ang, &s, &c);
    if (czf && qform_adj(czf, x)) {
        s = -s;
        c = -c;
    }
    return make_float2(float(c), float(s));
}

// Streaming observable step (n > 12) / forward-state readout.
// The seed factor 2 phase_O(t) D_f(t) conj(D_f(x)), t = x ^ X, factorises:
//   angle(x) = sum_{q in X} (x_q ? -w_q : w_q) = W_X - 2 sum_{q in X, x_q = 1} w_q,
//   CZ part  Q(x) ^ Q(x ^ X) = Q(X) ^ parity(x & M_X), M_X = xor of the adjacency
//            rows of X (Q quadratic, so its difference is affine),
// so a block (4096 amplitudes of one sample) builds e^{-2i w} products over the
// low 6 + 6 bits of x in two 64-entry tables and one constant for its high bits:
// per amplitude two table reads and two complex products instead of an fp64
// sincos (and no per-amplitude loops).
__global__ void __launch_bounds__(kThreads) seed_kernel(const SeedParams p) {
    const uint64_t dim = 1ull << p.n;
    const uint32_t per_block = dim < kTileAmps ? uint32_t(dim) : uint32_t(kTileAmps);
    const uint32_t chunks = uint32_t(dim / per_block);
    const uint32_t s = blockIdx.x / chunks, chunk = blockIdx.x % chunks;
    const float2 *psi = p.psi + s * dim;
    float2 *lam = p.lam + s * dim;
    if (p.apply_only) {
        for (uint32_t k = threadIdx.x; k < per_block; k += kThreads) {
            const uint32_t x = chunk * per_block + k;
            lam[x] = cmul(dfinal(x, p.n, p.wfinal, p.czfinal), psi[x]);
        }
        return;
    }
    __shared__ float2 t_lo[64], t_mid[64];
    __shared__ float2 c_blk;
    __shared__ uint32_t m_x, q_x;
    const uint32_t X = uint32_t(p.x_mask);
    const uint32_t xb = chunk * per_block; // high bits of x (low 12 bits are k)
    if (threadIdx.x < 128) {                // e^{-2i sum w} over bits 0..5 / 6..11 of x & X
        const int sh = threadIdx.x < 64 ? 0 : 6;
        const uint32_t v = (threadIdx.x & 63u) << sh;
        double a = 0.0;
        for (int q = sh; q < sh + 6 && q < p.n; ++q)
            if (((v & X) >> q) & 1u) a += p.wfinal[q];
        double sn, cs;
        sincos(-2.0 * a, &sn, &cs);
        (threadIdx.x < 64 ? t_lo : t_mid)[threadIdx.x & 63u] = make_float2(float(cs), float(sn));
    } else if (threadIdx.x == 128) {        // 2 i^y e^{i (W_X - 2 sum over the block's high bits)}
        double a = 0.0;
        for (int q = 0; q < p.n; ++q)
            if ((X >> q) & 1u) a += (q >= 12 && ((xb >> q) & 1u)) ? -p.wfinal[q] : p.wfinal[q];
        double sn, cs;
        sincos(a, &sn, &cs);
        double re = 2.0 * cs, im = 2.0 * sn, r2 = re, i2 = im;
        switch (p.y_count & 3u) {
        case 1: r2 = -im; i2 = re; break;
        case 2: r2 = -re; i2 = -im; break;
        case 3: r2 = im; i2 = -re; break;
        default: break;
        }
        c_blk = make_float2(float(r2), float(i2));
    } else if (threadIdx.x == 160) {        // CZ difference: Q(X) and M_X
        uint32_t m = 0, qx = 0;
        if (p.czfinal) {
            qx = qform_adj(p.czfinal, X);
            for (int q = 0; q < p.n; ++q) {
                if (!((X >> q) & 1u)) continue;
                uint32_t row = p.czfinal->adjlo[q]; // neighbours p < q ...
                for (int r = q + 1; r < p.n; ++r)   // ... and r > q
                    if ((p.czfinal->adjlo[r] >> q) & 1u) row |= 1u << r;
                m ^= row;
            }
        }
        m_x = m;
        q_x = qx;
    }
    __syncthreads();
    const float2 cb = c_blk;
    const uint32_t mx = m_x, qx = q_x, Z = uint32_t(p.z_mask);
    double e = 0.0;
    for (uint32_t k = threadIdx.x; k < per_block; k += kThreads) {
        const uint32_t x = xb + k, t = x ^ X;
        const uint32_t par = (__popc(t & Z) + qx + __popc(x & mx)) & 1u;
        const uint32_t xl = x & X;
        float2 f = cmul(cb, cmul(t_lo[xl & 63u], t_mid[(xl >> 6) & 63u]));
        if (par) f = make_float2(-f.x, -f.y);
        const float2 pt = psi[t], px = psi[x];
        const float2 l = cmul(f, pt);
        lam[x] = l;
        e += 0.5 * (double(px.x) * double(l.x) + double(px.y) * double(l.y));
    }
    __shared__ double red[kThreads / 32];
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) e += __shfl_xor_sync(0xffffffffu, e, m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) t += red[w];
        p.epart[size_t(s) * chunks + chunk] = t;
    }
}

// K accumulators per warp: [slots][12 local bits][8]. n < 12: 2 slots (stage
// parity); n = 12: a 4-slot ring by stage (the chained backward flushes stage s
// while stage s-1 is still accumulating, without a barrier of its own).
constexpr int res_kslots(bool n12) { return n12 ? 4 : 2; }
constexpr size_t res_acc(bool n12) { return size_t(8) * res_kslots(n12) * 12 * 8 * sizeof(double); }
// n = 12 reduces the expectation in registers (no per-amplitude fp64 scratch).
constexpr size_t res_es(bool n12) { return n12 ? 64 : size_t(kTileAmps) * sizeof(double); }
constexpr size_t res_smem(bool n12) {
    return size_t(2) * kTileBytes + res_es(n12) + 64 + 2 * 24 * 16 /*rys*/ + 2 * 16 * 8 /*treg*/ +
           2 * 6 * 8 /*mgs*/ + 64 /*kc, fold*/ + res_acc(n12) + 1024;
}

// N12: n == 12 (every group fully rotated): the phases are compile-time
// instances (no runtime group/ops dispatch), like the streaming passes' programs.
template <bool N12>
__global__ void __launch_bounds__(kThreads, 2)
    resident_kernel(const __grid_constant__ ResidentParams p,
                    const __grid_constant__ CUtensorMap m_psi0,
                    const __grid_constant__ CUtensorMap m_slots,
                    const __grid_constant__ CUtensorMap m_out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    uint8_t *pt = smem, *lt = smem + kTileBytes;
    double *es = reinterpret_cast<double *>(smem + 2 * kTileBytes);
    uint8_t *tail = smem + 2 * kTileBytes + res_es(N12);
    uint64_t *mbar = reinterpret_cast<uint64_t *>(tail);
    float4 *rys = reinterpret_cast<float4 *>(tail + 64);                  // [2 slots][24]
    float2 *treg_s = reinterpret_cast<float2 *>(tail + 64 + 2 * 24 * 16); // [2 slots][16]
    float2 *mgs = treg_s + 2 * 16;                                       // [2 slots][2][3]
    float *kc = reinterpret_cast<float *>(tail + 64 + 2 * 24 * 16 + 2 * 16 * 8 + 2 * 6 * 8); // [2][6]
    int *fold = reinterpret_cast<int *>(kc + 12);                                          // [2]
    double *acc = reinterpret_cast<double *>(tail + 64 + 2 * 24 * 16 + 2 * 16 * 8 + 2 * 6 * 8 + 64);
    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    const int n = p.n, S = p.stages;
    const uint32_t rot = (n >= 12) ? 0xFFFu : ((1u << n) - 1u);
    const uint32_t xmask = rot;
    const int spt = kTileAmps >> (n < 12 ? n : 12);

    constexpr int KS = res_kslots(N12);
    for (uint32_t i = tid; i < res_acc(N12) / 8; i += kThreads) acc[i] = 0.0;
    if (tid < 48) { // round-0 halves stay identity (t = 0, m = 1)
        rys[tid] = make_float4(0.f, 0.f, 1.f, 0.f);
    } else if (tid < 60) {
        mgs[tid - 48] = make_float2(1.f, 1.f);
    }
    if (tid == 0) {
        prefetch_map(&m_psi0);
        prefetch_map(&m_slots);
        mbar_init(&mbar[0], 1);
        fence_mbar_init();
    }
    __syncthreads();
    uint32_t phase = 0;
    // Stage data into slot s & 1 (threads 64..95). A stage is D_s then Ry_s on
    // groups 0, 1, 2; when the product F of its group scales is >= 2^-40 the
    // scales are folded into D_s (treg * F) and the Ry rounds run unscaled (the
    // tile is off by f in (F, 1] until the stage ends); the backward's K
    // measurements after undoing Ry_s on groups 2, 1, 0 then carry f^-2 and get
    // kc = (M2)^2, (M2 M1)^2, F^2 (qf_pass.cu pass_prologue, same algebra).
    auto load_stage = [&](int s) {
        const int sl = s & 1;
        auto gscale = [&](int g) {
            float M = 1.f;
            for (int b = 0; b < 4; ++b)
                if (4 * g + b < n) M *= ry_entry(p.ry[size_t(s) * n + 4 * g + b]).z;
            return M;
        };
        if (tid >= 64 && tid < 76) {
            const int lb = tid - 64;
            rys[sl * 24 + 12 + lb] = lb < n ? ry_entry(p.ry[size_t(s) * n + lb]) : make_float4(0.f, 0.f, 1.f, 0.f);
        } else if (tid >= 76 && tid < 92) {
            const float M0 = gscale(0), M1 = gscale(1), M2 = gscale(2), F = M0 * M1 * M2;
            float2 t = p.dt[s].treg[tid - 76];
            if (F >= 0x1p-40f) t = make_float2(t.x * F, t.y * F);
            treg_s[sl * 16 + (tid - 76)] = t;
            if (tid == 76) {
                const bool f = F >= 0x1p-40f;
                fold[sl] = f;
                kc[sl * 6 + 3 + 2] = f ? M2 * M2 : 1.f;
                kc[sl * 6 + 3 + 1] = f ? (M2 * M1) * (M2 * M1) : 1.f;
                kc[sl * 6 + 3 + 0] = f ? F * F : 1.f;
            }
        } else if (tid >= 92 && tid < 95) { // round-1 group scales
            const int g = tid - 92;
            const float M = gscale(g);
            mgs[sl * 6 + 3 + g] = make_float2(M, M);
        }
    };
    auto env_for = [&](int s) {
        PhaseEnv e;
        const int sl = s & 1;
        e.rys = rys + sl * 24;
        e.mgs = mgs + sl * 6;
        e.rot = rot;
        e.scale = !fold[sl];
        e.scale1 = e.scale;
        e.kc = kc + sl * 6;
        e.zm = s == 0 ? 3u : 0u; // Z at stage 0 only (zchain_kernel rebuilds the rest)
        e.treg_s = treg_s + sl * 16;
        e.acc_w = acc + warp * KS * 96;
        e.acc_w1 = e.acc_w + 12 * 8;
        const int c = p.stage_cz[s];
        const CzTab *cz = c >= 0 ? p.cztabs + c * p.cz_stride : nullptr;
        e.d = diag_ctx(tid, p.dt[s].tthr[tid], cz ? cz->thrinfo[tid] : 0u, p.dt + s, cz, nullptr, 0u);
        return e;
    };

    // ---- n = 12: chained stages, 2 shared-memory phases per stage instead of 3.
    // Stage s runs its Ry rounds on groups f(s), 1, l(s) with f(s) = 0 (s even) or
    // 2 (s odd) and l(s) = 2 - f(s); the phase that ends stage s-1 on group
    // l(s-1) = f(s) goes straight on with D_s and Ry_s there (the streaming
    // passes' pairing, qf_plan.cpp), split only where a checkpoint slot sits
    // between the two stages. D_s is tabulated in group f(s)'s orientation
    // (resident layouts 0 / 1, stage_layout = s & 1). Stage data live in a 4-entry
    // ring (stage s in entries s&1 and (s&1)+2), so the round-0 (stage a) and
    // round-1 (stage a+1) data of a phase are adjacent entries; K of stage s
    // accumulates in slot s&1. kc follows the stage's own group order.
    auto load12 = [&](int s) {
        const int e0 = s & 1, first = (s & 1) ? 2 : 0, last = 2 - first;
        auto gscale = [&](int g) {
            float M = 1.f;
            for (int b = 0; b < 4; ++b) M *= ry_entry(p.ry[size_t(s) * 12 + 4 * g + b]).z;
            return M;
        };
        if (tid >= 64 && tid < 76) {
            const int lb = tid - 64;
            const float4 v = ry_entry(p.ry[size_t(s) * 12 + lb]);
            rys[e0 * 12 + lb] = v;
            rys[(e0 + 2) * 12 + lb] = v;
        } else if (tid >= 76 && tid < 92) {
            const float M[3] = {gscale(0), gscale(1), gscale(2)};
            const float F = M[0] * M[1] * M[2];
            const bool f = F >= 0x1p-40f;
            float2 t = p.dt[s].treg[tid - 76];
            if (f) t = make_float2(t.x * F, t.y * F);
            treg_s[(s & 1) * 16 + (tid - 76)] = t;
            if (tid == 76) {
                for (int e = e0; e < 4; e += 2) {
                    fold[e] = f;
                    kc[e * 3 + last] = f ? M[last] * M[last] : 1.f;
                    kc[e * 3 + 1] = f ? (M[last] * M[1]) * (M[last] * M[1]) : 1.f;
                    kc[e * 3 + first] = f ? F * F : 1.f;
                }
            }
        } else if (tid >= 92 && tid < 95) {
            const int g = tid - 92;
            const float M = gscale(g);
            mgs[e0 * 3 + g] = make_float2(M, M);
            mgs[(e0 + 2) * 3 + g] = make_float2(M, M);
        }
    };
    // round 0 = stage a (a = -1: none), round 1 = stage a + 1, diagonal of stage d (-1: none)
    auto env12 = [&](int a, int d) {
        PhaseEnv e;
        const int b = a & 1;
        e.rys = rys + b * 12;
        e.mgs = mgs + b * 3;
        e.kc = kc + b * 3;
        e.rot = 0xFFFu;
        e.scale = !fold[b];
        e.scale1 = !fold[b + 1];
        e.zm = (a == 0 ? 1u : 0u) | (a + 1 == 0 ? 2u : 0u);
        e.acc_w = acc + warp * KS * 96 + (a & (KS - 1)) * 96;
        e.acc_w1 = acc + warp * KS * 96 + ((a + 1) & (KS - 1)) * 96;
        e.treg_s = treg_s + (d & 1) * 16;
        e.d.base = make_float2(1.f, 0.f);
        e.d.sgn = 0;
        if (d >= 0) {
            const int c = p.stage_cz[d];
            const CzTab *cz = c >= 0 ? p.cztabs + c * p.cz_stride + (d & 1) : nullptr;
            e.d = diag_ctx(tid, p.dt[d].tthr[tid], cz ? cz->thrinfo[tid] : 0u, p.dt + d, cz, nullptr, 0u);
        }
        return e;
    };
    auto slot_after = [&](int s) { // a checkpoint slot holds the state after stage s
        return ((s + 1) % p.ckpt == 0) && (s + 1 < S) && !p.forward_only;
    };

    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
        if (tid == 0) {
            mbar_expect_tx(&mbar[0], kTileBytes);
            tma_load3(pt, &m_psi0, &mbar[0], 0, t * 256, 0);
        }
        if (S > 0) {
            if constexpr (N12) load12(0);
            else load_stage(0);
        }
        mbar_wait(&mbar[0], phase);
        phase ^= 1u;
        __syncthreads();
        // ---------------- forward over all stages
        if constexpr (N12) {
            for (int s = 0; s < S; ++s) {
                const bool merged = s > 0 && !slot_after(s - 1);
                { // head: group f(s): [Ry_{s-1}] D_s Ry_s
                    const PhaseEnv e = env12(s - 1, s);
                    if (s & 1) {
                        if (merged) phase_fwd<2, 7u, true>(pt, tid, e);
                        else phase_fwd<2, 6u, true>(pt, tid, e);
                    } else {
                        if (merged) phase_fwd<0, 7u, true>(pt, tid, e);
                        else phase_fwd<0, 6u, true>(pt, tid, e);
                    }
                }
                __syncthreads();
                if (s + 1 < S) load12(s + 1); // stage s-1's ring entries are free now
                phase_fwd<1, 4u, true>(pt, tid, env12(s - 1, -1));
                __syncthreads();
                const bool slot = slot_after(s);
                if (s == S - 1 || slot) { // tail: Ry_s on group l(s) alone
                    const PhaseEnv e = env12(s - 1, -1);
                    if (s & 1) phase_fwd<0, 4u, true>(pt, tid, e);
                    else phase_fwd<2, 4u, true>(pt, tid, e);
                    if (slot) fence_async_smem();
                    __syncthreads();
                    if (slot) {
                        if (tid == 0) {
                            tma_store3(&m_slots, pt, 0, t * 256, (s + 1) / p.ckpt - 1);
                            bulk_commit();
                            bulk_wait_read0();
                        }
                        __syncthreads();
                    }
                }
            }
        } else {
            for (int s = 0; s < S; ++s) {
                const PhaseEnv e = env_for(s);
                if (s + 1 < S) load_stage(s + 1); // other slot: its latency overlaps this stage
                run_phase_fwd(0, pt, tid, 2u | 4u, e);
                __syncthreads();
                if (rot & 0xF0u) {
                    run_phase_fwd(1, pt, tid, 4u, e);
                    __syncthreads();
                }
                if (rot & 0xF00u) run_phase_fwd(2, pt, tid, 4u, e);
                const bool slot = slot_after(s);
                if (slot) fence_async_smem();
                __syncthreads();
                if (slot) {
                    if (tid == 0) {
                        tma_store3(&m_slots, pt, 0, t * 256, (s + 1) / p.ckpt - 1);
                        bulk_commit();
                        bulk_wait_read0();
                    }
                    __syncthreads();
                }
            }
        }
        if (p.forward_only) { // fold D_f and store the final state
#pragma unroll 4
            for (int j = 0; j < 16; ++j) {
                const uint32_t l = (tid << 4) | uint32_t(j);
                float2 *a = reinterpret_cast<float2 *>(pt + swz(l));
                *a = cmul(dfinal(l & xmask, n, p.wfinal, p.czfinal), *a);
            }
            fence_async_smem();
            __syncthreads();
            if (tid == 0) {
                tma_store3(&m_out, pt, 0, t * 256, 0);
                bulk_commit();
                bulk_wait_read0();
            }
            __syncthreads();
            continue;
        }
        // ---------------- observable: lambda = 2 O' psi, E per sample
        if constexpr (N12) { // one sample per tile: thread sums, warp butterfly, fixed warp order
            double e = 0.0;
#pragma unroll 4
            for (int j = 0; j < 16; ++j) {
                const uint32_t l = (tid << 4) | uint32_t(j);
                const uint32_t lp = l ^ uint32_t(p.x_mask);
                const float2 f = seed_factor(l, p.x_mask, p.z_mask, p.y_count, p.wfinal, p.czfinal);
                const float2 ps = *reinterpret_cast<const float2 *>(pt + swz(lp));
                const float2 px = *reinterpret_cast<const float2 *>(pt + swz(l));
                const float2 lv = cmul(f, ps);
                *reinterpret_cast<float2 *>(lt + swz(l)) = lv;
                e += 0.5 * (double(px.x) * double(lv.x) + double(px.y) * double(lv.y));
            }
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) e += __shfl_xor_sync(0xffffffffu, e, m);
            if ((tid & 31u) == 0) es[warp] = e;
            __syncthreads();
            if (tid == 0) {
                double sum = 0.0;
                for (int w = 0; w < 8; ++w) sum += es[w];
                if (uint32_t(t) < p.batch) p.expect[t] = sum;
            }
        } else {
#pragma unroll 4
            for (int j = 0; j < 16; ++j) {
                const uint32_t l = (tid << 4) | uint32_t(j);
                const uint32_t lp = l ^ uint32_t(p.x_mask);
                const float2 f = seed_factor(l & xmask, p.x_mask, p.z_mask, p.y_count, p.wfinal, p.czfinal);
                const float2 ps = *reinterpret_cast<const float2 *>(pt + swz(lp));
                const float2 px = *reinterpret_cast<const float2 *>(pt + swz(l));
                const float2 lv = cmul(f, ps);
                *reinterpret_cast<float2 *>(lt + swz(l)) = lv;
                es[l] = 0.5 * (double(px.x) * double(lv.x) + double(px.y) * double(lv.y));
            }
            __syncthreads();
            for (int st = 1; st < (1 << (n < 12 ? n : 12)); st <<= 1) {
                for (int i = tid; i < (kTileAmps >> 1) / st; i += kThreads) {
                    const int idx = i * 2 * st;
                    es[idx] += es[idx + st];
                }
                __syncthreads();
            }
            for (uint32_t ls = tid; ls < uint32_t(spt); ls += kThreads) { // n < 4: > 256 samples/tile
                const uint64_t sample = uint64_t(t) * spt + ls;
                if (sample < p.batch) p.expect[sample] = es[ls << (n < 12 ? n : 12)];
            }
        }
        // ---------------- backward
        // K of stage s from accumulator slot ks, added (RED) to this CTA's kpart row
        auto flush_k = [&](int s, int ks) {
            if (tid < 96) {
                const int lb = tid >> 3, c = tid & 7;
                if (lb < n) {
                    double sum = 0.0;
#pragma unroll
                    for (int w = 0; w < 8; ++w) {
                        double *a = acc + ((w * KS + ks) * 12 + lb) * 8 + c;
                        sum += *a;
                        *a = 0.0;
                    }
                    // fire-and-forget RED (no load round trip before the barrier); the
                    // slot is private to this CTA and this thread, so the adds stay in
                    // program order (deterministic)
                    atomicAdd(&p.kpart[(size_t(blockIdx.x) * S + s) * size_t(n) * 8 + lb * 8 + c], sum);
                }
            }
        };
        auto reanchor = [&](int s) { // psi := the forward state after stage s (slot)
            if (tid == 0) {
                mbar_expect_tx(&mbar[0], kTileBytes);
                tma_load3(pt, &m_slots, &mbar[0], 0, t * 256, (s + 1) / p.ckpt - 1);
            }
            mbar_wait(&mbar[0], phase);
            phase ^= 1u;
        };
        if constexpr (N12) {
            if (S > 0) load12(S - 1);
            __syncthreads();
            for (int s = S - 1; s >= 0; --s) {
                if (s == S - 1 || slot_after(s)) { // tail alone: undo Ry_s on group l(s)
                    if (slot_after(s)) reanchor(s);
                    const PhaseEnv e = env12(s - 1, -1);
                    if (s & 1) phase_bwd<0, 4u, true>(pt, lt, tid, e);
                    else phase_bwd<2, 4u, true>(pt, lt, tid, e);
                    __syncthreads();
                }
                if (s > 0) load12(s - 1); // stage s+1's ring entries are free now
                phase_bwd<1, 4u, true>(pt, lt, tid, env12(s - 1, -1));
                __syncthreads();
                { // head: group f(s): undo Ry_s, D_s [, Ry_{s-1}]
                    const bool merged = s > 0 && !slot_after(s - 1);
                    const PhaseEnv e = env12(s - 1, s);
                    if (s & 1) {
                        if (merged) phase_bwd<2, 7u, true>(pt, lt, tid, e);
                        else phase_bwd<2, 6u, true>(pt, lt, tid, e);
                    } else {
                        if (merged) phase_bwd<0, 7u, true>(pt, lt, tid, e);
                        else phase_bwd<0, 6u, true>(pt, lt, tid, e);
                    }
                }
                __syncthreads();
                // stage s is complete (its round-0 part came from iteration s + 1);
                // its ring slot is next written in iteration s - 3, barriers later
                flush_k(s, s & (KS - 1));
            }
            __syncthreads(); // the next tile reuses psi / lambda
        } else {
            if (S > 0) load_stage(S - 1);
            __syncthreads();
            for (int s = S - 1; s >= 0; --s) {
                if (slot_after(s)) reanchor(s);
                const PhaseEnv e = env_for(s);
                if (s > 0) load_stage(s - 1); // other slot: its latency overlaps this stage
                if (rot & 0xF00u) {
                    run_phase_bwd(2, pt, lt, tid, 4u, e);
                    __syncthreads();
                }
                if (rot & 0xF0u) {
                    run_phase_bwd(1, pt, lt, tid, 4u, e);
                    __syncthreads();
                }
                run_phase_bwd(0, pt, lt, tid, 4u | 2u, e);
                __syncthreads();
                flush_k(s, 1);
                __syncthreads();
            }
        }
    }
    if (tid == 0) bulk_wait0();
}

std::atomic<uint64_t> g_attrs{0};

} // namespace

size_t resident_smem_bytes() { return res_smem(true); }

int resident_occupancy() {
    const cudaError_t e = once_per_device(g_attrs, [] {
        cudaError_t r = cudaFuncSetAttribute(resident_kernel<false>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(res_smem(false)));
        if (r == cudaSuccess)
            r = cudaFuncSetAttribute(resident_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(res_smem(true)));
        return r;
    });
    if (e != cudaSuccess) return 0;
    int blocks = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, resident_kernel<false>, kThreads, res_smem(false));
    return blocks;
}

cudaError_t launch_resident(cudaStream_t st, int grid, const ResidentParams &p,
                            const CUtensorMap *psi0, const CUtensorMap *slots_map,
                            const CUtensorMap *out_map) {
    if (resident_occupancy() <= 0) return cudaErrorInvalidConfiguration;
    if (p.n == 12)
        resident_kernel<true><<<grid, kThreads, res_smem(true), st>>>(p, *psi0, *slots_map, *out_map);
    else
        resident_kernel<false><<<grid, kThreads, res_smem(false), st>>>(p, *psi0, *slots_map, *out_map);
    return cudaGetLastError();
}

cudaError_t launch_seed(cudaStream_t st, const SeedParams &p) {
    const uint64_t dim = 1ull << p.n;
    const uint64_t per_block = dim < kTileAmps ? dim : kTileAmps;
    const uint64_t blocks = (dim / per_block) * p.batch;
    seed_kernel<<<unsigned(blocks), kThreads, 0, st>>>(p);
    return cudaGetLastError();
}

} // namespace qfb
