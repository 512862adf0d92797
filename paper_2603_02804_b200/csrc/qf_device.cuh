// Device building blocks shared by the sm_100a kernels: PTX wrappers for
// TMA / mbarrier, tile addressing, the Ry / diagonal / K algebra on the
// 16 register-resident amplitudes of a group phase.
//
// Reference semantics restated (paths under /root/reference/proj):
//   fused forward of a block        engine.cpp:61-109 (composition fusion.cpp:127-152)
//   CZ parity sign                  engine.cpp:111-136
//   block backward Re<lam|du|psi>   engine.cpp:265-342
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "qf_internal.h"

namespace qfb {
namespace dev {

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t su32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile("{\n\t.reg .pred p;\n"
                 "WAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra WAIT_%=;\n}" ::"r"(su32(bar)),
                 "r"(parity)
                 : "memory");
}
__device__ __forceinline__ void tma_load5(void *dst, const CUtensorMap *map, uint64_t *bar, int c0,
                                          int c1, int c2, int c3, int c4) {
    asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(dst)),
                 "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
                 "r"(c4), "r"(su32(bar))
                 : "memory");
}
// L2 prefetch of a 5-D tile (no shared memory, no completion tracking).
__device__ __forceinline__ void tma_prefetch5(const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                              int c4) {
    asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
                 : "memory");
}
__device__ __forceinline__ void tma_store5(const CUtensorMap *map, const void *src, int c0, int c1,
                                           int c2, int c3, int c4) {
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group"
                 " [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(su32(src))
                 : "memory");
}
__device__ __forceinline__ void tma_load3(void *dst, const CUtensorMap *map, uint64_t *bar, int c0,
                                          int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(su32(dst)),
                 "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void tma_store3(const CUtensorMap *map, const void *src, int c0, int c1,
                                           int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group"
                 " [%0, {%1, %2, %3}], [%4];" ::"l"(reinterpret_cast<uint64_t>(map)), "r"(c0),
                 "r"(c1), "r"(c2), "r"(su32(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;"); }
__device__ __forceinline__ void bulk_wait_read0() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap *m) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
// Align a dynamic-smem pointer to 1024 B (SWIZZLE_128B) by pointer arithmetic
// on the shared pointer itself, so the compiler keeps the shared address space
// (LDS/STS, not generic LD/ST).
__device__ __forceinline__ uint8_t *align1024(uint8_t *p) {
    return p + ((1024u - (su32(p) & 1023u)) & 1023u);
}

// ------------------------------------------------------- tile addressing
// Byte offset of register j of thread tau in group phase G. 16-B chunk c of
// row r lives at chunk c ^ (r & 7) (SWIZZLE_128B); every phase's LDS/STS
// pattern is bank-conflict free (G0 as 16-B pairs, G1/G2 as 8-B words).
template <int G> __device__ __forceinline__ uint32_t goff(uint32_t tau, int j) {
    if (G == 0) {
        return (tau << 7) | (((uint32_t(j >> 1) ^ tau) & 7u) << 4) | (uint32_t(j & 1) << 3);
    } else if (G == 1) {
        return ((tau >> 4) << 11) | (uint32_t(j) << 7) |
               (((((tau & 15u) >> 1) ^ uint32_t(j)) & 7u) << 4) | ((tau & 1u) << 3);
    } else {
        return (uint32_t(j) << 11) | ((tau >> 4) << 7) |
               (((((tau & 15u) >> 1) ^ (tau >> 4)) & 7u) << 4) | ((tau & 1u) << 3);
    }
}
__device__ __forceinline__ uint32_t swz(uint32_t l) {
    const uint32_t r = l >> 4, c = l & 15u;
    return (r << 7) | ((((c >> 1) ^ r) & 7u) << 4) | ((c & 1u) << 3);
}
// Explicit shared-space accesses (LDS/STS) on 32-bit shared addresses, so no
// code path can fall back to generic LD/ST.
__device__ __forceinline__ float2 lds64(uint32_t a) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ float4 lds128(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(a));
    return v;
}
__device__ __forceinline__ void sts64(uint32_t a, float2 v) {
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
}
template <int G>
__device__ __forceinline__ void lds16(const uint8_t *tile, uint32_t tau, float2 (&v)[16]) {
    const uint32_t base = su32(tile);
    if (G == 0) {
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
            const float4 t = lds128(base + goff<0>(tau, j));
            v[j] = make_float2(t.x, t.y);
            v[j + 1] = make_float2(t.z, t.w);
        }
    } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = lds64(base + goff<G>(tau, j));
    }
}
template <int G>
__device__ __forceinline__ void sts16(uint8_t *tile, uint32_t tau, const float2 (&v)[16]) {
    const uint32_t base = su32(tile);
    if (G == 0) {
#pragma unroll
        for (int j = 0; j < 16; j += 2)
            sts128(base + goff<0>(tau, j), make_float4(v[j].x, v[j].y, v[j + 1].x, v[j + 1].y));
    } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) sts64(base + goff<G>(tau, j), v[j]);
    }
}

// ------------------------------------------------------ packed complex math
// Blackwell FFMA2/FMUL2: two fp32 lanes per issue. A complex64 amplitude is
// one register pair, so real-coefficient updates vectorise over (re, im).
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) { // conj(a) * b
    return make_float2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
// The same products as one FMUL2 + one FFMA2 (the (v.y, v.x) operand is a free
// register-pair swizzle): g v = (g.x, g.x) v + (-g.y, g.y) swap(v).
#ifndef QF_DIAG2
#define QF_DIAG2 1
#endif
__device__ __forceinline__ float2 cmul_p(float2 g, float2 v) {
    return f2fma(make_float2(-g.y, g.y), make_float2(v.y, v.x), f2mul(make_float2(g.x, g.x), v));
}
__device__ __forceinline__ float2 cmulc_p(float2 g, float2 v) { // conj(g) v
    return f2fma(make_float2(g.y, -g.y), make_float2(v.y, v.x), f2mul(make_float2(g.x, g.x), v));
}

// Ry(beta) = [[c, -s], [s, c]] (circuit.cpp:67-68) on register bit B, with c
// factored out: Ry = c [[1, -t], [t, 1]], t = s / c, so the bit costs ONE FFMA2
// per output amplitude; the c of the group's four bits are re-applied together
// (one FMUL2 per amplitude, ry_round). fp32 rounding of fma(-t, b, a) * c is
// the same relative error as c a - s b; c is clamped at 2^-20 (beta ~ pi) so
// intermediates stay < 2^80 x |amplitude| (error <= 1e-6 relative, only there).
// rys entry: (t, t, c, 0). Backward applies Ry(-beta): t -> -t.
template <int B, bool INV>
__device__ __forceinline__ void ry2(float2 (&v)[16], float4 e) {
    const float2 K = make_float2(e.x, e.y);
    const float2 N = make_float2(-e.x, -e.y);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        if (j & (1 << B)) continue;
        const float2 a = v[j], b = v[j | (1 << B)];
        v[j] = f2fma(INV ? K : N, b, a);             // a -/+ t b
        v[j | (1 << B)] = f2fma(INV ? N : K, a, b);  // b +/- t a
    }
}
// One Ry round on the rotated bits of group G, then the product of their m
// (mg = (M, M)) unless the pass folds every scale of its two rounds into its
// diagonal (scale == false, pass_prologue). FULL (all four bits rotated, the
// HEA case) has no per-bit branches around the register array; otherwise
// warp-uniform branches.
template <int G, bool INV, bool FULL>
__device__ __forceinline__ void ry_round(float2 (&v)[16], const float4 *rys, uint32_t rot,
                                         float2 mg, bool scale) {
    if (FULL || (rot & (1u << (4 * G + 0)))) ry2<0, INV>(v, rys[4 * G + 0]);
    if (FULL || (rot & (1u << (4 * G + 1)))) ry2<1, INV>(v, rys[4 * G + 1]);
    if (FULL || (rot & (1u << (4 * G + 2)))) ry2<2, INV>(v, rys[4 * G + 2]);
    if (FULL || (rot & (1u << (4 * G + 3)))) ry2<3, INV>(v, rys[4 * G + 3]);
    if (scale) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = f2mul(mg, v[j]);
    }
}
// (cos, sin) of beta/2 -> rys entry; the group scale is the product of m.
__device__ __forceinline__ float4 ry_entry(float2 cs) {
    const float c = fmaxf(cs.x, 0x1.0p-20f); // cos(beta/2) >= 0 (beta in [0, pi])
    const float t = cs.y / c;
    return make_float4(t, t, c, 0.f);
}

// Gradient data of register bit B. Every reference gradient of the qubit's
// section is (1/2) sum_m R_m Im Tr(sigma_m K) with K = sum psi lam^dag (the
// generators only ever appear conjugated by unitaries, finalize_kernel), so
// three real numbers per (stage, qubit) suffice:
//   X = Im(K01 + K10),  Y = Re(K01 - K10),  Z = Im(K00 - K11).
// With ps = swap(psi) (a free operand swizzle of FFMA2):
// (ps (.) lam).x - .y = Im(psi conj lam), (psi (.) lam).x + .y = Re(psi conj lam).
// 6 FFMA2 per pair into ONE accumulator per output (measured 29 vs 24 TFMA/s
// for two interleaved sets, tools/ffma2_patterns.cu); the four bits of a
// group give 12 independent chains.
template <int B, bool WZ>
__device__ __forceinline__ void kbit3(const float2 (&p)[16], const float2 (&l)[16], float *out) {
    float2 bx = make_float2(0.f, 0.f), ay = bx, bz = bx;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        if (j & (1 << B)) continue;
        const int j1 = j | (1 << B);
        const float2 ps0 = make_float2(p[j].y, p[j].x), ps1 = make_float2(p[j1].y, p[j1].x);
        if (WZ) bz = f2fma(ps0, l[j], bz);
        bx = f2fma(ps0, l[j1], bx);
        ay = f2fma(p[j], l[j1], ay);
        ay = f2fma(make_float2(-p[j1].x, -p[j1].y), l[j], ay);
        bx = f2fma(ps1, l[j], bx);
        if (WZ) bz = f2fma(make_float2(-ps1.x, -ps1.y), l[j1], bz);
    }
    out[0] = bx.x - bx.y;
    out[1] = ay.x + ay.y;
    if (WZ) out[2] = bz.x - bz.y;
}

// All four register bits at once, lambda-major: the 12 FFMA2 that read l[j]
// run back to back, so l[j] stays in the operand reuse cache and each FFMA2
// fetches two fresh register pairs (three would cost a third issue cycle;
// measured 30.8 vs 29.0 TFMA/s, tools/ffma2_patterns.cu). 12 accumulators,
// each updated every 12th instruction.
template <bool WZ>
__device__ __forceinline__ void kbit3_all(const float2 (&p)[16], const float2 (&l)[16], float *out) {
    constexpr int C = WZ ? 3 : 2; // outputs per bit: X, Y (, Z)
    float2 r[12];
#pragma unroll
    for (int i = 0; i < 12; ++i) r[i] = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int k = j ^ (1 << b);
            const float2 psj = make_float2(p[j].y, p[j].x), psk = make_float2(p[k].y, p[k].x);
            float2 &bx = r[C * b], &ay = r[C * b + 1], &bz = r[C * b + C - 1];
            if (!(j & (1 << b))) { // l[j] = lambda_0 of the pair
                if (WZ) bz = f2fma(psj, l[j], bz);
                bx = f2fma(psk, l[j], bx);
                ay = f2fma(make_float2(-p[k].x, -p[k].y), l[j], ay);
            } else {               // l[j] = lambda_1 of the pair
                if (WZ) bz = f2fma(make_float2(-psj.x, -psj.y), l[j], bz);
                bx = f2fma(psk, l[j], bx);
                ay = f2fma(p[k], l[j], ay);
            }
        }
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        out[C * b + 0] = r[C * b].x - r[C * b].y;
        out[C * b + 1] = r[C * b + 1].x + r[C * b + 1].y;
        if (WZ) out[C * b + 2] = r[C * b + 2].x - r[C * b + 2].y;
    }
}

// (X, Y, Z) of the rotated bits of group G at the current point: 12 values
// reduced over the warp in one 16-wide reduce-scatter (16 shuffles), then
// added in fp64 (times kc, the pass's scale correction) to this warp's
// accumulator acc_w[local bit][8] (slots 0..2).
//
// WZ = false measures only (X, Y) (8 values, 9 shuffles): Z commutes with the
// diagonals and with every gate on other qubits, so Z before Ry_s(q) equals Z
// just after Ry_{s-1}(q) = cos(b) Z_{s-1} - sin(b) X_{s-1} (b = beta_{s-1}(q)),
// rebuilt per qubit by zchain_kernel; only stage 0 measures Z.
//
// kslot != nullptr (compiled backward programs, (X, Y) only): the reduce-scatter
// stops at 8-lane groups and each lane adds its value (index lane & 7, times kc)
// to a per-thread fp32 register accumulator that lives across tiles
// (kreg_flush at the end of the kernel), instead of an fp64 shared-memory
// read-modify-write per tile.
template <int G, bool FULL, bool WZ>
__device__ __forceinline__ void kmeasure(const float2 (&p)[16], const float2 (&l)[16],
                                         uint32_t rot, double *acc_w, float kc,
                                         float *kslot = nullptr) {
#if QF_ABLATE_K
    return; // timing ablation only
#endif
    constexpr int C = WZ ? 3 : 2;
    constexpr int NV = WZ ? 16 : 8; // reduce width
    float v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = 0.f;
    if (FULL) {
        kbit3_all<WZ>(p, l, v);
    } else {
        if (rot & (1u << (4 * G + 0))) kbit3<0, WZ>(p, l, v + 0 * C);
        if (rot & (1u << (4 * G + 1))) kbit3<1, WZ>(p, l, v + 1 * C);
        if (rot & (1u << (4 * G + 2))) kbit3<2, WZ>(p, l, v + 2 * C);
        if (rot & (1u << (4 * G + 3))) kbit3<3, WZ>(p, l, v + 3 * C);
    }
    const uint32_t lane = threadIdx.x & 31u;
#pragma unroll
    for (int m = NV / 2; m >= 1; m >>= 1) {
        const bool up = (lane & m) != 0;
#pragma unroll
        for (int i = 0; i < m; ++i) {
            const float send = up ? v[i] : v[i + m];
            const float keep = up ? v[i + m] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
        }
    }
    if (!WZ && kslot) {
        *kslot = fmaf(v[0], kc, *kslot);
        return;
    }
    float r = v[0];
#pragma unroll
    for (int m = NV; m < 32; m <<= 1) r += __shfl_xor_sync(0xffffffffu, r, m);
    if (lane < uint32_t(4 * C)) {
        const uint32_t bit = lane / uint32_t(C), comp = lane % uint32_t(C);
        if (rot & (1u << (4 * G + bit))) acc_w[(4 * G + bit) * 8 + comp] += double(r) * double(kc);
    }
}

// narrow_to_bf16 (statevec.hpp:36-45): round to nearest even, NaN quieted
__device__ __forceinline__ uint32_t bf16_rne_bits(float v) {
    const uint32_t u = __float_as_uint(v);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (u >> 16) | 0x0040u;
    return (u + 0x7fffu + ((u >> 16) & 1u)) >> 16;
}

// ------------------------------------------------------------- diagonal
__device__ __forceinline__ uint32_t linmask4(uint32_t M) {
    uint32_t m = 0;
    if (M & 1u) m ^= 0xAAAAu;
    if (M & 2u) m ^= 0xCCCCu;
    if (M & 4u) m ^= 0xF0F0u;
    if (M & 8u) m ^= 0xFF00u;
    return m;
}
struct DiagCtx {
    float2 base;  // e^{i phi(thread bits, tile bits)}
    uint32_t sgn; // bit j: sign flip of register j
};
// tthr / thrinfo are per-thread constants of a launch; tile terms per tile.
__device__ __forceinline__ DiagCtx diag_ctx(uint32_t tau, float2 tthr, uint32_t thrinfo,
                                            const DiagTab *dt, const CzTab *cz,
                                            const uint32_t *tileinfo, uint32_t tb) {
    DiagCtx d;
    float2 b = tthr;
    if (tb) b = cmul(b, cmul(dt->tt1[tb & 255u], dt->tt2[(tb >> 8) & 255u]));
    d.base = b;
    d.sgn = 0;
    if (cz) {
        const uint32_t ti = tileinfo ? tileinfo[tb] : 0u;
        const uint32_t sbase = (ti ^ (thrinfo >> 4) ^ __popc(tau & (ti >> 8))) & 1u;
        d.sgn = (sbase ? 0xFFFFu : 0u) ^ cz->qreg ^ linmask4(((ti >> 1) ^ thrinfo) & 15u);
    }
    return d;
}
template <bool CONJ>
__device__ __forceinline__ void apply_diag(float2 (&v)[16], const DiagCtx &d, const float2 *treg_s) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        float2 g = cmul(d.base, treg_s[j]);
        const uint32_t flip = (d.sgn << (31 - j)) & 0x80000000u;
        g.x = __uint_as_float(__float_as_uint(g.x) ^ flip);
        g.y = __uint_as_float(__float_as_uint(g.y) ^ flip);
        // packed products only in the forward (measured: forward -2%, backward +2%
        // with packed products: register pressure of the psi + lambda phases)
        if (QF_DIAG2 && !CONJ) v[j] = cmul_p(g, v[j]);
        else v[j] = CONJ ? cmulc(g, v[j]) : cmul(g, v[j]);
    }
}

// ---------------------------------------------------------- group phases
struct PhaseEnv {
    const float4 *rys; // smem [2][12] ry_entry(): round 0, round 1
    const float2 *mgs; // smem [2][3] group scales (M, M): round 0, round 1
    uint32_t rot;
    bool scale;        // round 0: apply the group scales (false: folded into the diagonal)
    bool scale1;       // the same for round 1 (rounds of two stages may differ)
    DiagCtx d;
    const float2 *treg_s;
    const float *kc;   // smem [2][3] K scale corrections (nullptr = 1)
    uint32_t zm;       // bit r: round r measures Z (stage 0 only; zchain_kernel)
    double *acc_w;     // this warp's [12][8] accumulators of round 0
    double *acc_w1;    // ... and of round 1
    float *kreg;       // compiled backward programs: per-thread [2 rounds][3 groups]
};
__device__ __forceinline__ float kcorr(const PhaseEnv &e, int r, int g) {
    return e.kc ? e.kc[3 * r + g] : 1.f;
}
// OPS: 1 = round 0, 2 = diagonal, 4 = round 1 (compile-time, so the 16-register
// arrays stay in place across the whole phase).
template <int G, uint32_t OPS, bool FULL>
__device__ __forceinline__ void phase_fwd(uint8_t *tile, uint32_t tau, const PhaseEnv &e) {
    float2 v[16];
    lds16<G>(tile, tau, v);
    if (OPS & 1u) ry_round<G, false, FULL>(v, e.rys, e.rot, e.mgs[G], e.scale);
    if (OPS & 2u) apply_diag<false>(v, e.d, e.treg_s);
    if (OPS & 4u) ry_round<G, false, FULL>(v, e.rys + 12, e.rot, e.mgs[3 + G], e.scale1);
    sts16<G>(tile, tau, v);
}
template <int G, uint32_t OPS, bool FULL, bool RTZ = true>
__device__ __forceinline__ void phase_bwd(uint8_t *pt, uint8_t *lt, uint32_t tau, const PhaseEnv &e) {
    float2 p[16], l[16];
#if QF_ABLATE_SMEM // timing ablation only: no shared-memory traffic in the phases
#pragma unroll
    for (int j = 0; j < 16; ++j) p[j] = l[j] = make_float2(float(tau + j), 1.f);
#else
    lds16<G>(pt, tau, p);
    lds16<G>(lt, tau, l);
#endif
#if QF_ABLATE_MATH // timing ablation only: shared-memory traffic without the math
    sts16<G>(pt, tau, p);
    sts16<G>(lt, tau, l);
    return;
#endif
    if (OPS & 4u) {
        ry_round<G, true, FULL>(p, e.rys + 12, e.rot, e.mgs[3 + G], e.scale1);
        ry_round<G, true, FULL>(l, e.rys + 12, e.rot, e.mgs[3 + G], e.scale1);
        if (RTZ && (e.zm & 2u)) kmeasure<G, FULL, true>(p, l, e.rot, e.acc_w1, kcorr(e, 1, G));
        else kmeasure<G, FULL, false>(p, l, e.rot, e.acc_w1, kcorr(e, 1, G), RTZ ? nullptr : e.kreg + 3 + G);
    }
    if (OPS & 2u) {
        apply_diag<true>(p, e.d, e.treg_s);
        apply_diag<true>(l, e.d, e.treg_s);
    }
    if (OPS & 1u) {
        ry_round<G, true, FULL>(p, e.rys, e.rot, e.mgs[G], e.scale);
        ry_round<G, true, FULL>(l, e.rys, e.rot, e.mgs[G], e.scale);
        if (RTZ && (e.zm & 1u)) kmeasure<G, FULL, true>(p, l, e.rot, e.acc_w, kcorr(e, 0, G));
        else kmeasure<G, FULL, false>(p, l, e.rot, e.acc_w, kcorr(e, 0, G), RTZ ? nullptr : e.kreg + G);
    }
#if QF_ABLATE_SMEM
    if (p[0].x == 1.2345f && l[3].y == 5.4321f) sts16<G>(pt, tau, p); // keep the math live
#else
    sts16<G>(pt, tau, p);
    sts16<G>(lt, tau, l);
#endif
}

// Runtime (group, ops, full) -> template instance. ops in {1, 4, 2|4, 1|2|4}.
template <int G, bool FULL>
__device__ __forceinline__ void run_fwd_g(uint32_t ops, uint8_t *tile, uint32_t tau,
                                          const PhaseEnv &e) {
    switch (ops) {
    case 1: phase_fwd<G, 1, FULL>(tile, tau, e); break;
    case 4: phase_fwd<G, 4, FULL>(tile, tau, e); break;
    case 6: phase_fwd<G, 6, FULL>(tile, tau, e); break;
    default: phase_fwd<G, 7, FULL>(tile, tau, e); break;
    }
}
template <int G, bool FULL>
__device__ __forceinline__ void run_bwd_g(uint32_t ops, uint8_t *pt, uint8_t *lt, uint32_t tau,
                                          const PhaseEnv &e) {
    switch (ops) {
    case 1: phase_bwd<G, 1, FULL>(pt, lt, tau, e); break;
    case 4: phase_bwd<G, 4, FULL>(pt, lt, tau, e); break;
    case 6: phase_bwd<G, 6, FULL>(pt, lt, tau, e); break;
    default: phase_bwd<G, 7, FULL>(pt, lt, tau, e); break;
    }
}
__device__ __forceinline__ void run_phase_fwd(int g, uint8_t *tile, uint32_t tau, uint32_t ops,
                                              const PhaseEnv &e) {
    const bool full = ((e.rot >> (4 * g)) & 0xFu) == 0xFu;
    if (g == 0) full ? run_fwd_g<0, true>(ops, tile, tau, e) : run_fwd_g<0, false>(ops, tile, tau, e);
    else if (g == 1) full ? run_fwd_g<1, true>(ops, tile, tau, e) : run_fwd_g<1, false>(ops, tile, tau, e);
    else full ? run_fwd_g<2, true>(ops, tile, tau, e) : run_fwd_g<2, false>(ops, tile, tau, e);
}
__device__ __forceinline__ void run_phase_bwd(int g, uint8_t *pt, uint8_t *lt, uint32_t tau,
                                              uint32_t ops, const PhaseEnv &e) {
    const bool full = ((e.rot >> (4 * g)) & 0xFu) == 0xFu;
    if (g == 0) full ? run_bwd_g<0, true>(ops, pt, lt, tau, e) : run_bwd_g<0, false>(ops, pt, lt, tau, e);
    else if (g == 1) full ? run_bwd_g<1, true>(ops, pt, lt, tau, e) : run_bwd_g<1, false>(ops, pt, lt, tau, e);
    else full ? run_bwd_g<2, true>(ops, pt, lt, tau, e) : run_bwd_g<2, false>(ops, pt, lt, tau, e);
}

// ------------------------------------------------ compile-time phase programs
// A pass's phase list as a constant, so the common passes (HEA interior passes
// of layouts A and B) run as one straight-line sequence of inlined phases with
// no runtime dispatch: bits 0..2 nph, bits 3..5 FULL per group, phase i at bit
// 6 + 5i: group (2 bits), ops (3 bits). Encoded on the host by prog_encode.
constexpr uint32_t prog_nph(uint32_t P) { return P & 7u; }
constexpr bool prog_full(uint32_t P, int g) { return (P >> (3 + g)) & 1u; }
constexpr int prog_g(uint32_t P, int i) { return int((P >> (6 + 5 * i)) & 3u); }
constexpr uint32_t prog_ops(uint32_t P, int i) { return (P >> (8 + 5 * i)) & 7u; }

// Groups 0 and 1 place the same local bits (9..11) in the warp index (goff),
// so between two such phases each warp reads only what it wrote: sync receives
// std::integral_constant<bool, cross_warp> and may use __syncwarp.
constexpr bool prog_cross(int ga, int gb) { return ga == 2 || gb == 2; }

// Backward: phases I, I-1, ..., 0 with sync(cross) between them; no Z measurement.
template <uint32_t P, int I, class Sync>
__device__ __forceinline__ void prog_bwd(uint8_t *pt, uint8_t *lt, uint32_t tau, const PhaseEnv &e,
                                         Sync &&sync) {
    if constexpr (I >= 0) {
        constexpr int g = prog_g(P, I);
        phase_bwd<g, prog_ops(P, I), prog_full(P, g), false>(pt, lt, tau, e);
        if constexpr (I > 0) {
            sync(std::integral_constant<bool, prog_cross(g, prog_g(P, I - 1))>{});
            prog_bwd<P, I - 1>(pt, lt, tau, e, sync);
        }
    }
}
// Forward: phases I, I+1, ..., nph-1.
template <uint32_t P, int I, class Sync>
__device__ __forceinline__ void prog_fwd(uint8_t *tile, uint32_t tau, const PhaseEnv &e, Sync &&sync) {
    if constexpr (I < int(prog_nph(P))) {
        constexpr int g = prog_g(P, I);
        phase_fwd<g, prog_ops(P, I), prog_full(P, g)>(tile, tau, e);
        if constexpr (I + 1 < int(prog_nph(P))) {
            sync(std::integral_constant<bool, prog_cross(g, prog_g(P, I + 1))>{});
            prog_fwd<P, I + 1>(tile, tau, e, sync);
        }
    }
}

} // namespace dev
} // namespace qfb
