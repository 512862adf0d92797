// Forward pass of layout A with 64-amplitude register groups.
//
// The interior forward passes of layout A (all 12 local qubits rotated twice,
// the stage diagonal between: Ry_{s-1}(A) -> D_s -> Ry_s(A))
// take five shared-memory phases with the 4-bit groups of qf_pass.cu. Here a
// thread holds 6 local bits (64 amplitudes, 128 registers; the forward carries
// psi only), so the pass is THREE phases:
//     H(round 0)  ->  L(round 0, D, round 1)  ->  H(round 1)
// with  L = local bits {0,1,2,3,7,8},  H = {4,5,6,9,10,11}  (qf_internal.h).
// The split keeps every LDS/STS conflict-free on the TMA 128B-swizzled tile: in
// an L phase the lanes vary local bits 4..6 (row bits 0..2, i.e. the 8 swizzle
// patterns of a 16-B chunk), in an H phase a warp reads 2 whole 128-B rows.
// Shared-memory traffic per tile: 3 x 64 KiB + the TMA 64 KiB (was 5 x 64 + 64).
//
// A *team* of 64 threads (2 warps) owns one tile at a time; T teams per CTA
// (one CTA per SM) share a ring of NB = 7 tile buffers, so NB - T tiles are in
// flight while T are transformed: tile k of the CTA is team k % T's, lives in
// buffer k % NB, completes mbarrier k % NB (parity (k / NB) & 1). The team that
// stores tile k reloads its buffer with tile k + NB one phase later (its
// store's shared-memory read has finished by then).
//
// Numerics are the narrow kernel's: Ry = c [[1, -t], [t, 1]] with one FFMA2 per
// output amplitude, the group scales folded into the diagonal when their product
// F >= 2^-40 (qf_pass.cu pass_prologue), the diagonal as base(tile, thread) x
// treg(j) with CZ signs from the wide tables.
#include "qf_device.cuh"

namespace qfb {
namespace {

using namespace dev;

constexpr int kTeam = 64;
constexpr int kWideNB = 7;

// local index of register j (6 bits) of thread tau (6 bits) in group G
// (0 = L: j -> {0,1,2,3,7,8}, tau -> {4,5,6,9,10,11}; 1 = H: the other way round)
template <int G> __device__ __forceinline__ uint32_t wlocal(uint32_t tau, uint32_t j) {
    const uint32_t a = G == 0 ? j : tau; // bits of local {0,1,2,3,7,8}
    const uint32_t b = G == 0 ? tau : j; // bits of local {4,5,6,9,10,11}
    return (a & 15u) | (((a >> 4) & 3u) << 7) | ((b & 7u) << 4) | (((b >> 3) & 7u) << 9);
}

template <int G>
__device__ __forceinline__ void wlds(const uint8_t *tile, uint32_t tau, float2 (&v)[64]) {
    const uint32_t base = su32(tile);
    if (G == 0) {
#pragma unroll
        for (int j = 0; j < 64; j += 2) {
            const float4 t = lds128(base + swz(wlocal<0>(tau, uint32_t(j))));
            v[j] = make_float2(t.x, t.y);
            v[j + 1] = make_float2(t.z, t.w);
        }
    } else {
#pragma unroll
        for (int j = 0; j < 64; ++j) v[j] = lds64(base + swz(wlocal<1>(tau, uint32_t(j))));
    }
}
template <int G>
__device__ __forceinline__ void wsts(uint8_t *tile, uint32_t tau, const float2 (&v)[64]) {
    const uint32_t base = su32(tile);
    if (G == 0) {
#pragma unroll
        for (int j = 0; j < 64; j += 2)
            sts128(base + swz(wlocal<0>(tau, uint32_t(j))), make_float4(v[j].x, v[j].y, v[j + 1].x, v[j + 1].y));
    } else {
#pragma unroll
        for (int j = 0; j < 64; ++j) sts64(base + swz(wlocal<1>(tau, uint32_t(j))), v[j]);
    }
}

// Ry on register bit B of the 64 amplitudes (forward): 32 pairs, one FFMA2 per output.
template <int B> __device__ __forceinline__ void wry(float2 (&v)[64], float4 e) {
    const float2 K = make_float2(e.x, e.y);
    const float2 N = make_float2(-e.x, -e.y);
#pragma unroll
    for (int j = 0; j < 64; ++j) {
        if (j & (1 << B)) continue;
        const float2 a = v[j], b = v[j | (1 << B)];
        v[j] = f2fma(N, b, a);
        v[j | (1 << B)] = f2fma(K, a, b);
    }
}
// One Ry round on the 6 register bits of group G (all rotated in layout A).
// rys: [12] entries of the round, by local bit.
template <int G>
__device__ __forceinline__ void wround(float2 (&v)[64], const float4 *rys, float2 mg, bool scale) {
    wry<0>(v, rys[G == 0 ? 0 : 4]);
    wry<1>(v, rys[G == 0 ? 1 : 5]);
    wry<2>(v, rys[G == 0 ? 2 : 6]);
    wry<3>(v, rys[G == 0 ? 3 : 9]);
    wry<4>(v, rys[G == 0 ? 7 : 10]);
    wry<5>(v, rys[G == 0 ? 8 : 11]);
    if (scale) {
#pragma unroll
        for (int j = 0; j < 64; ++j) v[j] = f2mul(mg, v[j]);
    }
}

__device__ __forceinline__ unsigned long long linmask6(uint32_t M) {
    unsigned long long m = 0;
    if (M & 1u) m ^= 0xAAAAAAAAAAAAAAAAull;
    if (M & 2u) m ^= 0xCCCCCCCCCCCCCCCCull;
    if (M & 4u) m ^= 0xF0F0F0F0F0F0F0F0ull;
    if (M & 8u) m ^= 0xFF00FF00FF00FF00ull;
    if (M & 16u) m ^= 0xFFFF0000FFFF0000ull;
    if (M & 32u) m ^= 0xFFFFFFFF00000000ull;
    return m;
}

__device__ __forceinline__ void wdiag(float2 (&v)[64], float2 base, unsigned long long sgn,
                                      const float2 *treg_s) {
#pragma unroll
    for (int j = 0; j < 64; ++j) {
        float2 g = cmul(base, treg_s[j]);
        const uint32_t flip = uint32_t(sgn >> j) << 31;
        g.x = __uint_as_float(__float_as_uint(g.x) ^ flip);
        g.y = __uint_as_float(__float_as_uint(g.y) ^ flip);
#if QF_DIAG2
        v[j] = cmul_p(g, v[j]);
#else
        v[j] = cmul(g, v[j]);
#endif
    }
}

__device__ __forceinline__ void team_bar(int id) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kTeam) : "memory");
}

constexpr size_t wide_smem() {
    return size_t(kWideNB) * kTileBytes + 64 /*mbar*/ + 24 * 16 /*rys*/ + 64 * 8 /*treg*/ +
           4 * 8 /*mgs*/ + 1024 /*align*/;
}

template <int T>
__global__ void __launch_bounds__(T * kTeam, 1)
    pass_fwd_wide(const __grid_constant__ PassParams p, const __grid_constant__ CUtensorMap m_in,
                  const __grid_constant__ CUtensorMap m_out) {
    static_assert(T >= 1 && T < kWideNB, "ring needs a spare buffer");
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    uint8_t *tail = smem + kWideNB * kTileBytes;
    uint64_t *mbar = reinterpret_cast<uint64_t *>(tail);
    float4 *rys = reinterpret_cast<float4 *>(tail + 64);            // [2 rounds][12 local bits]
    float2 *treg_s = reinterpret_cast<float2 *>(tail + 64 + 24 * 16); // [64]
    float2 *mgs = treg_s + 64;                                        // [2 rounds][L, H]
    const uint32_t tid = threadIdx.x, team = tid / kTeam, tau = tid % kTeam;

    const int lo_mask = (1 << p.tile_lo_bits) - 1, hi_mask = (1 << p.tile_hi_bits) - 1;
    const int sample_shift = p.tile_lo_bits + p.tile_hi_bits;
    const uint32_t tis_mask = (1u << sample_shift) - 1u;
    const int stride = gridDim.x;
    auto tile_of = [&](int k) { return int(blockIdx.x) + k * stride; };
    auto issue_load = [&](int k) {
        const int t = tile_of(k);
        const int c1 = t & lo_mask, c3 = (t >> p.tile_lo_bits) & hi_mask, c4 = t >> sample_shift;
        uint64_t *bar = &mbar[k % kWideNB];
        mbar_expect_tx(bar, kTileBytes);
        tma_load5(smem + (k % kWideNB) * kTileBytes, &m_in, bar, 0, c1, 0, c3, c4);
    };
    if (tid == 0) {
        prefetch_map(&m_in);
        prefetch_map(&m_out);
        for (int b = 0; b < kWideNB; ++b) mbar_init(&mbar[b], 1);
        fence_mbar_init();
        for (int k = 0; k < kWideNB; ++k)
            if (tile_of(k) < p.tiles) issue_load(k);
    }
    // stage data: Ry entries by local bit, group scales, the diagonal's register table
    if (tid < 24) {
        const int r = tid / 12, lb = tid % 12;
        const int s = r == 0 ? p.s0 : p.s1;
        rys[tid] = ry_entry(p.ry[size_t(s) * p.n + p.qmap[lb]]);
    } else if (tid >= 32 && tid < 36) {
        const int r = (tid - 32) / 2, g = (tid - 32) % 2;
        const int s = r == 0 ? p.s0 : p.s1;
        float M = 1.f;
        for (int b = 0; b < 6; ++b) {
            const int lb = g == 0 ? wide_reg_bit(b) : wide_thr_bit(b);
            M *= ry_entry(p.ry[size_t(s) * p.n + p.qmap[lb]]).z;
        }
        mgs[tid - 32] = make_float2(M, M);
    }
    __syncthreads();
    const float F = mgs[0].x * mgs[1].x * mgs[2].x * mgs[3].x;
    const bool fold = F >= 0x1p-40f;
    for (uint32_t j = tid; j < 64; j += blockDim.x) {
        float2 t = p.dtw->treg[j];
        if (fold) t = make_float2(t.x * F, t.y * F);
        treg_s[j] = t;
    }
    __syncthreads();
    const bool scale = !fold;
    const float2 tthr = p.dtw->tthr[tau];
    const uint32_t thrinfo = p.czw ? p.czw->thrinfo[tau] : 0u;
    const unsigned long long qreg = p.czw ? p.czw->qreg : 0ull;
    const int bar_id = 1 + int(team);

    int pending = -1; // tile whose load this team's leader still owes (deferred refill)
    auto refill = [&] {
        if (tau == 0 && pending >= 0) {
            bulk_wait_read0();
            issue_load(pending);
            pending = -1;
        }
    };
    for (int k = int(team); tile_of(k) < p.tiles; k += T) {
        const int t = tile_of(k);
        if (p.l2pf & 2) refill(); // early refill: the store's smem read (~0.1 us) is done by now
        // diagonal inputs of this tile, loaded now and combined after the first phase
        const uint32_t tb = uint32_t(t) & tis_mask;
        const float2 t1 = p.dt->tt1[tb & 255u], t2 = p.dt->tt2[(tb >> 8) & 255u];
        const uint32_t ti = (p.czw && p.tileinfow) ? p.tileinfow[tb] : 0u;
        mbar_wait(&mbar[k % kWideNB], (k / kWideNB) & 1);
        uint8_t *pt = smem + (k % kWideNB) * kTileBytes;
        float2 v[64];
        // H: round 0
        wlds<1>(pt, tau, v);
        wround<1>(v, rys, mgs[1], scale);
        wsts<1>(pt, tau, v);
        team_bar(bar_id);
        if (!(p.l2pf & 2)) refill();
        // L: round 0, D, round 1 (the diagonal's inputs were loaded before the first phase)
        {
            const float2 base = tb ? cmul(tthr, cmul(t1, t2)) : tthr;
            unsigned long long sgn = 0;
            if (p.czw) {
                const uint32_t sbase = (ti ^ (thrinfo >> 6) ^ __popc(tau & (ti >> 8))) & 1u;
                sgn = (sbase ? ~0ull : 0ull) ^ qreg ^ linmask6(((ti >> 1) ^ thrinfo) & 63u);
            }
            wlds<0>(pt, tau, v);
            wround<0>(v, rys, mgs[0], scale);
            wdiag(v, base, sgn, treg_s);
            wround<0>(v, rys + 12, mgs[2], scale);
            wsts<0>(pt, tau, v);
        }
        team_bar(bar_id);
        // H: round 1
        wlds<1>(pt, tau, v);
        wround<1>(v, rys + 12, mgs[3], scale);
        wsts<1>(pt, tau, v);
        fence_async_smem();
        team_bar(bar_id);
        if (p.slot16) {
            // StorageMode::MemSave slot pass: the tile's bf16 copy straight from shared
            // memory (narrow_to_bf16, statevec.hpp:36-45), instead of a narrow kernel
            // re-reading the state (layout A: the tile is amplitudes [4096 t, 4096 t + 4096))
            uint4 *dst = reinterpret_cast<uint4 *>(p.slot16 + size_t(t) * kTileAmps);
            const uint32_t base = su32(pt);
#pragma unroll 4
            for (uint32_t i = 0; i < uint32_t(kTileAmps) / (4 * kTeam); ++i) {
                const uint32_t q = i * kTeam + tau, l = 4 * q;
                const float4 a = lds128(base + swz(l)), b = lds128(base + swz(l + 2));
                dst[q] = make_uint4(bf16_rne_bits(a.x) | (bf16_rne_bits(a.y) << 16),
                                    bf16_rne_bits(a.z) | (bf16_rne_bits(a.w) << 16),
                                    bf16_rne_bits(b.x) | (bf16_rne_bits(b.y) << 16),
                                    bf16_rne_bits(b.z) | (bf16_rne_bits(b.w) << 16));
            }
        }
        if (tau == 0) {
            const int c1 = t & lo_mask, c3 = (t >> p.tile_lo_bits) & hi_mask, c4 = t >> sample_shift;
            tma_store5(&m_out, pt, 0, c1, 0, c3, c4);
            bulk_commit();
            if (tile_of(k + kWideNB) < p.tiles) pending = k + kWideNB;
        }
    }
    if (tau == 0) {
        if (pending >= 0) { // the team's last tile: nobody else owes this load
            bulk_wait_read0();
            issue_load(pending);
        }
        bulk_wait0();
    }
}

#ifndef QF_WIDE_TEAMS
#define QF_WIDE_TEAMS 4
#endif
constexpr int kWideTeams = QF_WIDE_TEAMS;
std::atomic<uint64_t> g_wide_attr{0};

} // namespace

int wide_grid(int sms) { return sms; }

cudaError_t launch_pass_wide(cudaStream_t st, int grid, const PassParams &p, const CUtensorMap *psi_in,
                             const CUtensorMap *psi_out) {
    const cudaError_t e = once_per_device(g_wide_attr, [] {
        return cudaFuncSetAttribute(pass_fwd_wide<kWideTeams>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(wide_smem()));
    });
    if (e != cudaSuccess) return e;
    pass_fwd_wide<kWideTeams><<<grid, kWideTeams * kTeam, wide_smem(), st>>>(p, *psi_in, *psi_out);
    return cudaGetLastError();
}

} // namespace qfb
