// complex128 fused path: the reference's double instantiations
// (gradient<double> engine.cpp:716-755, run_checkpointed<double>
// checkpoint.cpp:144-163, instantiated at engine.cpp:942 / checkpoint.cpp:196-213)
// with one HBM pass per *segment* instead of one per gate.
//
// Ops (build_c128_plan): a section = a maximal run of consecutive rotations on
// one qubit, applied as ONE 2x2 unitary U (the rotations multiplied in fp64,
// later gates on the left, like compose_block_unitary fusion.cpp:127-152); a
// CZ run = one diagonal sign (apply_cz_kernel engine.cpp:111-136); a CNOT =
// a conditional pair swap (apply_cnot_kernel engine.cpp:142-170). A segment is
// a range of ops whose non-diagonal targets fit one tile of 2^m amplitudes in
// shared memory (m = min(n, 11); qubits 0..2 always local so every 8
// amplitudes are one 128-B line): one HBM pass. One CTA loads a tile (psi, and
// lambda in the backward) and runs the segment's *rounds* on it: a round holds
// up to three sections on (at most) three local bits plus the CZ runs between
// them, applied to the eight amplitudes of those bits in each thread's
// registers (one shared-memory read and write per round); a CNOT is a round of
// its own (pair swaps in shared memory).
//
// Backward: for each section, in reverse, psi_in = U^dag psi_out and lam_in =
// U^dag lam_out (psi uncomputed in place: unitary in fp64, the same choice as
// the per-gate c128 path). The gradient of rotation j of the section is
//   Re <lam_out| A_j dg_j B_j |psi_in> = Re Tr(M_j K),  K = sum_pairs psi_in lam_in^dag,
// M_j = B_j^dag g_j^dag dg_j B_j (B_j = the rotations before j; rotation_derivative
// circuit.cpp:76-87). With dg = -(i/2) P g, M_j = -(i/2) H_j, H_j = sum_m h_m sigma_m
// hermitian and traceless, so Re Tr(M_j K) = (1/2)(hx X + hy Y + hz Z) with
//   X = Im(K01 + K10), Y = Re(K01 - K10), Z = Im(K00 - K11):
// three accumulators per section (12 FMA per pair instead of 16), evaluated in
// fp64 by c128_finalize. K partials are reduced per warp, per CTA in fixed warp
// order, and over CTAs in fixed order by the last CTA of the segment:
// deterministic.
#include <algorithm>
#include <functional>
#include <set>
#include <stdexcept>

#include "qf_internal.h"

namespace qfb {
namespace {

constexpr int kT = 256; // threads per CTA

struct Cx2 { // 2x2 complex, row-major [[a, b], [c, d]]
    double2 a, b, c, d;
};
__device__ __forceinline__ double2 cm(double2 x, double2 y) {
    return make_double2(x.x * y.x - x.y * y.y, x.x * y.y + x.y * y.x);
}
__device__ __forceinline__ double2 cadd(double2 x, double2 y) { return make_double2(x.x + y.x, x.y + y.y); }
__device__ __forceinline__ double2 cj(double2 x) { return make_double2(x.x, -x.y); }
__device__ __forceinline__ Cx2 mul(const Cx2 &x, const Cx2 &y) {
    return {cadd(cm(x.a, y.a), cm(x.b, y.c)), cadd(cm(x.a, y.b), cm(x.b, y.d)),
            cadd(cm(x.c, y.a), cm(x.d, y.c)), cadd(cm(x.c, y.b), cm(x.d, y.d))};
}
__device__ __forceinline__ Cx2 dag(const Cx2 &x) { return {cj(x.a), cj(x.c), cj(x.b), cj(x.d)}; }
__device__ __forceinline__ Cx2 ident() {
    return {make_double2(1, 0), make_double2(0, 0), make_double2(0, 0), make_double2(1, 0)};
}
// u = c I - i s P (rotation_matrix, circuit.cpp:61-73); with (c, s) ->
// (-s/2, c/2) the same formula is the derivative (circuit.cpp:76-87).
__device__ __forceinline__ Cx2 rot(int axis, double c, double s) {
    const double2 z = make_double2(0, 0);
    if (axis == 0) return {make_double2(c, 0), make_double2(0, -s), make_double2(0, -s), make_double2(c, 0)};
    if (axis == 1) return {make_double2(c, 0), make_double2(-s, 0), make_double2(s, 0), make_double2(c, 0)};
    return {make_double2(c, -s), z, z, make_double2(c, s)};
}

// Per section: U (the rotations multiplied in fp64, later gates on the left, like
// compose_block_unitary fusion.cpp:127-152), then U = e^{i d} Rz(a) Ry(b) Rz(g) in
// fp64 and the round data of it (kC128SecWords double2):
//   [0] (p, q): Ry(b) = m [[p, -q], [q, p]] with (p, q) = (1, tan b/2), m = cos b/2
//       when cos >= sin, else (cot b/2, 1), m = sin b/2 (two DFMA per output either way)
//   [1] (m, g)   [2], [3] e^{-ig/2}, e^{+ig/2}   [4], [5] e^{id} e^{-ia/2}, e^{id} e^{+ia/2}
__global__ void c128_prep(int nsec, const uint32_t *off, const uint32_t *cnt, const uint32_t *gates,
                          const double *theta, double2 *secU) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nsec) return;
    Cx2 U = ident();
    for (uint32_t i = 0; i < cnt[s]; ++i) {
        const uint32_t g = gates[off[s] + i];
        double sn, cs;
        sincos(theta[g >> 2] / 2.0, &sn, &cs);
        U = mul(rot(int(g & 3u), cs, sn), U);
    }
    const double2 det = cadd(cm(U.a, U.d), make_double2(-(U.b.x * U.c.x - U.b.y * U.c.y),
                                                        -(U.b.x * U.c.y + U.b.y * U.c.x)));
    const double d = 0.5 * atan2(det.y, det.x);
    double sd, cd;
    sincos(-d, &sd, &cd);
    const double2 ph = make_double2(cd, sd);             // e^{-id}
    const double2 a = cm(ph, U.a), b = cm(ph, U.c);      // V = e^{-id} U in SU(2): V00, V10
    const double c = hypot(a.x, a.y), sn = hypot(b.x, b.y);
    const double arga = c > 0.0 ? atan2(a.y, a.x) : 0.0, argb = sn > 0.0 ? atan2(b.y, b.x) : 0.0;
    const double al = argb - arga, ga = -arga - argb;    // a + g = -2 arg V00, a - g = 2 arg V10
    double2 *w = secU + size_t(s) * kC128SecWords;
    if (c >= sn) {
        w[0] = make_double2(1.0, sn / c);
        w[1] = make_double2(c, ga);
    } else {
        w[0] = make_double2(c / sn, 1.0);
        w[1] = make_double2(sn, ga);
    }
    double sg, cg, sa, ca;
    sincos(0.5 * ga, &sg, &cg);
    sincos(0.5 * al, &sa, &ca);
    w[2] = make_double2(cg, -sg);
    w[3] = make_double2(cg, sg);
    const double2 ed = make_double2(cd, -sd);            // e^{+id}
    w[4] = cm(ed, make_double2(ca, -sa));
    w[5] = cm(ed, make_double2(ca, sa));
}

// K per section: (X, Y, Z); grad of rotation j = (1/2)(hx X + hy Y + hz Z) with
// H_j = B_j^dag g_j^dag P_j g_j B_j = [[hz, hx - i hy], [hx + i hy, -hz]].
__global__ void c128_finalize(int nsec, const uint32_t *off, const uint32_t *cnt,
                              const uint32_t *gates, const double *theta, const double2 *secU,
                              const double *K, double *grad) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nsec) return;
    const double X = K[size_t(s) * 3 + 0], Y = K[size_t(s) * 3 + 1], Z = K[size_t(s) * 3 + 2];
    // K was measured after the section's Rz(g) (the rounds apply all Rz(g) of a round
    // first): K' = G K G^dag, G = Rz(g), so Re Tr(M K) = Re Tr(G M G^dag K')
    const double gam = secU[size_t(s) * kC128SecWords + 1].y;
    double sg, cg;
    sincos(0.5 * gam, &sg, &cg);
    const Cx2 G = {make_double2(cg, -sg), make_double2(0, 0), make_double2(0, 0), make_double2(cg, sg)};
    Cx2 B = ident();
    for (uint32_t i = 0; i < cnt[s]; ++i) {
        const uint32_t g = gates[off[s] + i];
        const int axis = int(g & 3u);
        double sn, cs;
        sincos(theta[g >> 2] / 2.0, &sn, &cs);
        const Cx2 u = rot(axis, cs, sn), P = rot(axis, 0.0, 1.0); // rot(axis, 0, 1) = -i P
        const Cx2 uB = mul(u, B);
        const Cx2 H = mul(G, mul(mul(dag(uB), mul(P, uB)), dag(G))); // = -i G B^dag g^dag P g B G^dag
        // H holds -i H_j: hz = Re H_j00 = -Im H00, hx + i hy = H_j10 = i H10
        const double hz = -H.a.y, hx = -H.c.y, hy = H.c.x;
        grad[g >> 2] = 0.5 * (hx * X + hy * Y + hz * Z);
        B = uB;
    }
}

// Shared-memory slot of tile amplitude l: the low 3 bits (the 16-B bank group of a
// complex128) XORed with the fold of the higher 3-bit chunks, so a quarter-warp's
// eight 16-B accesses are conflict-free whenever its threads vary local bits whose
// positions are distinct mod 3 (the round planner prefers such octets).
__device__ __forceinline__ uint32_t sw2(uint32_t l) {
    return l ^ (((l >> 3) ^ (l >> 6) ^ (l >> 9)) & 7u);
}

__device__ __forceinline__ uint32_t insert0(uint32_t p, uint32_t pos) {
    return ((p >> pos) << (pos + 1)) | (p & ((1u << pos) - 1u));
}

__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gmem_src) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Unscaled Ry on register bit B: forward R'(p, q) = [[p, -q], [q, p]], inverse R'(p, -q);
// (p, q) = (1, t) (fa) or (t', 1): one DFMA per output component.
template <int B, int R, bool INV>
__device__ __forceinline__ void ry_bit(bool fa, double2 pq, double2 (&v)[1 << R]) {
    const double t = fa ? pq.y : pq.x;
#pragma unroll
    for (int j = 0; j < (1 << R); ++j) {
        if (j & (1 << B)) continue;
        const double2 a = v[j], b = v[j | (1 << B)];
        if (fa) { // a' = a -+ t b, b' = b +- t a
            const double tt = INV ? t : -t;
            v[j] = make_double2(fma(tt, b.x, a.x), fma(tt, b.y, a.y));
            v[j | (1 << B)] = make_double2(fma(-tt, a.x, b.x), fma(-tt, a.y, b.y));
        } else { // forward a' = t a - b, b' = a + t b; inverse a' = t a + b, b' = t b - a
            v[j] = INV ? make_double2(fma(t, a.x, b.x), fma(t, a.y, b.y))
                       : make_double2(fma(t, a.x, -b.x), fma(t, a.y, -b.y));
            v[j | (1 << B)] = INV ? make_double2(fma(t, b.x, -a.x), fma(t, b.y, -a.y))
                                  : make_double2(fma(t, b.x, a.x), fma(t, b.y, a.y));
        }
    }
}
// (X, Y, Z) of register bit B: X += Im(a lb* + b la*), Y += Re(a lb* - b la*),
// Z += Im(a la* - b lb*)   (a, b = psi of the pair, la, lb = lambda)
template <int B, int R>
__device__ __forceinline__ void kacc_bit(double *k, const double2 (&v)[1 << R], const double2 (&w)[1 << R]) {
#pragma unroll
    for (int j = 0; j < (1 << R); ++j) {
        if (j & (1 << B)) continue;
        const double2 a = v[j], b = v[j | (1 << B)], la = w[j], lb = w[j | (1 << B)];
        k[0] = fma(a.y, lb.x, fma(-a.x, lb.y, fma(b.y, la.x, fma(-b.x, la.y, k[0]))));
        k[1] = fma(a.x, lb.x, fma(a.y, lb.y, fma(-b.x, la.x, fma(-b.y, la.y, k[1]))));
        k[2] = fma(a.y, la.x, fma(-a.x, la.y, fma(-b.y, lb.x, fma(b.x, lb.y, k[2]))));
    }
}

constexpr int kWarps = kT / 32;
// K slot s (runtime) -> accumulator row (compile-time indices: no local memory)
template <int B, int R>
__device__ __forceinline__ void kacc_slot(uint32_t slot, double (&kk)[kC128RoundSecs][3],
                                          const double2 (&v)[1 << R], const double2 (&w)[1 << R]) {
    if (slot == 0) kacc_bit<B, R>(kk[0], v, w);
    else if (slot == 1) kacc_bit<B, R>(kk[1], v, w);
    else kacc_bit<B, R>(kk[2], v, w);
}

template <bool BWD, int R>
__global__ void __launch_bounds__(kT, 2) seg_c128(const C128Seg sg, const C128Op *__restrict__ ops,
                                               const C128Round *__restrict__ rounds,
                                               const uint32_t *__restrict__ czp,
                                               const double2 *__restrict__ secU, double2 *psi,
                                               double2 *lam, int n, uint64_t tiles, double *kpart,
                                               unsigned *ticket, double *K) {
    extern __shared__ double2 sm[];
    const uint32_t m = sg.m, amps = 1u << m;
    double2 *sp = sm, *sl = sm + amps;
    // round tables: [round][16] = Dg[8] (all Rz(g) of the round), Da'[8] (all Rz(a),
    // the global phases and the Ry scales m), then [round][4] K scales; then K slots
    double2 *rtab = sm + (BWD ? 2u : 1u) * amps;
    double *kscl = reinterpret_cast<double *>(rtab + size_t(kC128MaxRounds) * 16);
    double *acc = kscl + size_t(kC128MaxRounds) * 4; // [sec][warp][3]
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
    __shared__ int8_t lpos[32];
    __shared__ uint8_t lq[16], rq[32];
    __shared__ C128Op ops_s[kC128MaxOps];
    __shared__ C128Round rnd_s[kC128MaxRounds];
    __shared__ double2 u_s[kC128MaxSec * kC128SecWords];
    __shared__ uint32_t cz_s[kC128MaxCzPairs];
    if (tid == 0) { // constant indices: no local copy of the parameter block
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            lpos[i] = sg.lpos[i];
            rq[i] = sg.rq[i];
            if (i < 16) lq[i] = sg.lq[i];
        }
    }
    const uint32_t nops = sg.op_end - sg.op_begin, nrnd = sg.round_end - sg.round_begin;
    for (uint32_t i = tid; i < nops; i += kT) ops_s[i] = ops[sg.op_begin + i];
    for (uint32_t i = tid; i < nrnd; i += kT) rnd_s[i] = rounds[sg.round_begin + i];
    for (uint32_t i = tid; i < sg.nsec * kC128SecWords; i += kT)
        u_s[i] = secU[size_t(sg.sec_begin) * kC128SecWords + i];
    for (uint32_t i = tid; i < sg.cz_count; i += kT) cz_s[i] = czp[sg.cz_begin + i];
    if (BWD)
        for (uint32_t i = tid; i < sg.nsec * kWarps * 3; i += kT) acc[i] = 0.0;
    __syncthreads();
    for (uint32_t w = tid; w < nrnd * 16; w += kT) { // Dg / Da' entries of every round
        const C128Round rd = rnd_s[w >> 4];
        if (rd.kind != 0) continue;
        const uint32_t j = w & 7u, alpha = (w >> 3) & 1u;
        double2 f = make_double2(1.0, 0.0);
        for (uint32_t k = 0; k < rd.nsec; ++k) {
            const double2 *u = u_s + rd.sec[k] * kC128SecWords;
            const uint32_t bit = (j >> rd.sbit[k]) & 1u;
            f = cm(f, u[(alpha ? 4 : 2) + bit]);
            if (alpha) f = make_double2(f.x * u[1].x, f.y * u[1].x);
        }
        rtab[w] = f;
        if (j == 0 && !alpha) { // K slot k is measured with psi, lambda off by f = prod_{l<k} m_l
            double sc = 1.0;    // (the scales of the slots not undone yet): K carries f^2
            for (uint32_t k = 0; k < rd.nsec; ++k) {
                kscl[(w >> 4) * 4 + k] = sc;
                const double m = u_s[rd.sec[k] * kC128SecWords + 1].x;
                sc /= m * m;
            }
        }
    }
    __syncthreads();
    constexpr int KA = (1 << kC128TileBits) / kT; // tile amplitudes per thread (copy in / out)
    // local part of their global index (recomputed at the copies: fewer live registers
    // through the rounds)
    uint32_t xla[KA];
#pragma unroll
    for (int k = 0; k < KA; ++k) {
        const uint32_t l = tid + uint32_t(k) * kT;
        uint32_t x = 0;
        for (uint32_t j = 0; j < m; ++j) x |= ((l >> j) & 1u) << lq[j];
        xla[k] = x;
    }
    auto xl = [&](int k) { return xla[k]; };
    auto tile_xr = [&](uint64_t t) {
        const uint32_t r = uint32_t(t) & ((1u << sg.nrest) - 1u);
        uint32_t xr = 0;
        for (uint32_t k = 0; k < sg.nrest; ++k) xr |= ((r >> k) & 1u) << rq[k];
        return xr;
    };
    constexpr int NV = 1 << R;
    for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const uint64_t base = (t >> sg.nrest) << n;
        const uint32_t xr = tile_xr(t);
#pragma unroll
        for (int k = 0; k < KA; ++k) {
            const uint32_t l = tid + uint32_t(k) * kT;
            if (l < amps) {
                const uint32_t x = xr | xl(k);
                cp_async16(sp + sw2(l), psi + base + x);
                if (BWD) cp_async16(sl + sw2(l), lam + base + x);
            }
        }
        cp_async_commit();
        cp_async_wait_all();
        __syncthreads();
        for (uint32_t ri = 0; ri < nrnd; ++ri) {
            const uint32_t rix = BWD ? nrnd - 1 - ri : ri;
            const C128Round rd = rnd_s[rix];
            if (rd.kind == 1) { // CNOT(control a, target q): pair swaps, self-inverse
                const C128Op op = ops_s[rd.op_begin - sg.op_begin];
                const uint32_t pos = uint32_t(lpos[op.q]);
                const int cpos = lpos[op.a];
                for (uint32_t p = tid; p < (amps >> 1); p += kT) {
                    const uint32_t i0 = insert0(p, pos), i1 = i0 | (1u << pos);
                    const uint32_t ctl = cpos >= 0 ? (i0 >> cpos) & 1u : (xr >> op.a) & 1u;
                    if (ctl) {
                        double2 tmp = sp[sw2(i0)];
                        sp[sw2(i0)] = sp[sw2(i1)];
                        sp[sw2(i1)] = tmp;
                        if (BWD) {
                            tmp = sl[sw2(i0)];
                            sl[sw2(i0)] = sl[sw2(i1)];
                            sl[sw2(i1)] = tmp;
                        }
                    }
                }
            } else {
                double kk[kC128RoundSecs][3];
#pragma unroll
                for (int s2 = 0; s2 < kC128RoundSecs; ++s2) kk[s2][0] = kk[s2][1] = kk[s2][2] = 0.0;
                if (tid < (amps >> R)) {
                    uint32_t bl = tid; // local index of register offset 0
#pragma unroll
                    for (int i = 0; i < R; ++i) bl = insert0(bl, rd.bits[i]);
                    // shared-memory slot of register offset j (recomputed at the store:
                    // fewer live registers than keeping eight addresses)
                    auto slot = [&](int j) {
                        uint32_t o = 0;
#pragma unroll
                        for (int i = 0; i < R; ++i) o |= uint32_t((j >> i) & 1) << rd.bits[i];
                        return sw2(bl | o);
                    };
                    double2 v[NV], w[NV];
#pragma unroll
                    for (int j = 0; j < NV; ++j) {
                        const uint32_t a = slot(j);
                        v[j] = sp[a];
                        if (BWD) w[j] = sl[a];
                    }
                    uint32_t x0 = 0; // global index of register offset 0 (CZ runs only)
                    if (rd.has_cz) {
                        x0 = xr;
                        for (uint32_t j = 0; j < m; ++j) x0 |= ((bl >> j) & 1u) << lq[j];
                    }
                    // e^{id} Rz(a) Ry(b) Rz(g) per section: all Rz(g) of the round first (Dg),
                    // the unscaled Ry (two DFMA per output), all Rz(a), phases and Ry scales last
                    // (Da'); CZ runs in place. The backward runs the inverse: conj(Da') (the
                    // scales m stay in it: R'^-1 = m^2 R'(p, -q)), R'(p, -q), conj(Dg).
                    const double2 *tb = rtab + size_t(rix) * 16;
                    if (BWD) {
#pragma unroll
                        for (int j = 0; j < NV; ++j) {
                            const double2 f = cj(tb[8 + j]);
                            v[j] = cm(f, v[j]);
                            w[j] = cm(f, w[j]);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < NV; ++j) v[j] = cm(tb[j], v[j]);
                    }
                    const uint32_t no = rd.op_end - rd.op_begin;
                    for (uint32_t oi = 0; oi < no; ++oi) {
                        const C128Op op = ops_s[(BWD ? rd.op_end - 1 - oi : rd.op_begin + oi) - sg.op_begin];
                        if (op.type == 0) {
                            const double2 pq = u_s[(op.a - sg.sec_begin) * kC128SecWords];
                            const bool fa = pq.x == 1.0; // (1, tan) form, else (cot, 1)
                            if (op.q == 0) {
                                ry_bit<0, R, BWD>(fa, pq, v);
                                if (BWD) { ry_bit<0, R, BWD>(fa, pq, w); kacc_slot<0, R>(op.b, kk, v, w); }
                            } else if (R > 1 && op.q == 1) {
                                ry_bit<(R > 1 ? 1 : 0), R, BWD>(fa, pq, v);
                                if (BWD) { ry_bit<(R > 1 ? 1 : 0), R, BWD>(fa, pq, w); kacc_slot<(R > 1 ? 1 : 0), R>(op.b, kk, v, w); }
                            } else if (R > 2) {
                                ry_bit<(R > 2 ? 2 : 0), R, BWD>(fa, pq, v);
                                if (BWD) { ry_bit<(R > 2 ? 2 : 0), R, BWD>(fa, pq, w); kacc_slot<(R > 2 ? 2 : 0), R>(op.b, kk, v, w); }
                            }
                        } else { // CZ run: Q(x0 | o) = Q(x0) ^ Q(o) ^ parity(o & M(x0))
                            uint32_t qx = 0, M = 0;
                            for (uint32_t c = 0; c < op.b; ++c) {
                                const uint32_t pr = cz_s[op.a - sg.cz_begin + c], a = pr & 255u, b = pr >> 8;
                                const uint32_t ra = (x0 >> a) & 1u, rb = (x0 >> b) & 1u;
                                qx ^= ra & rb;
                                M ^= (ra << b) ^ (rb << a);
                            }
                            uint32_t mr = 0;
#pragma unroll
                            for (int i = 0; i < R; ++i) mr |= ((M >> rd.gq[i]) & 1u) << i;
#pragma unroll
                            for (int j = 0; j < NV; ++j) {
                                if ((qx ^ (op.q >> j) ^ __popc(uint32_t(j) & mr)) & 1u) {
                                    v[j] = make_double2(-v[j].x, -v[j].y);
                                    if (BWD) w[j] = make_double2(-w[j].x, -w[j].y);
                                }
                            }
                        }
                    }
                    if (BWD) {
#pragma unroll
                        for (int j = 0; j < NV; ++j) {
                            const double2 f = cj(tb[j]);
                            v[j] = cm(f, v[j]);
                            w[j] = cm(f, w[j]);
                        }
#pragma unroll
                        for (int s2 = 0; s2 < kC128RoundSecs; ++s2) { // Ry scales still applied at K
                            const double f = kscl[rix * 4 + s2];
                            kk[s2][0] *= f;
                            kk[s2][1] *= f;
                            kk[s2][2] *= f;
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < NV; ++j) v[j] = cm(tb[8 + j], v[j]);
                    }
#pragma unroll
                    for (int j = 0; j < NV; ++j) {
                        const uint32_t a = slot(j);
                        sp[a] = v[j];
                        if (BWD) sl[a] = w[j];
                    }
                }
                if (BWD) { // warp sums of the round's (X, Y, Z): one 16-wide reduce-scatter
                    // (15 shuffles + 1) instead of a butterfly per value (45); lane l < 9 ends
                    // with value l = 3 slot + component and adds it to this warp's slot
                    double r[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) r[i] = i < 9 ? kk[i / 3][i % 3] : 0.0;
#pragma unroll
                    for (int mm = 8; mm >= 1; mm >>= 1) {
                        const bool up = (lane & uint32_t(mm)) != 0;
#pragma unroll
                        for (int i = 0; i < mm; ++i) {
                            const double send = up ? r[i] : r[i + mm];
                            const double keep = up ? r[i + mm] : r[i];
                            r[i] = keep + __shfl_xor_sync(0xffffffffu, send, mm);
                        }
                    }
                    const double x = r[0] + __shfl_xor_sync(0xffffffffu, r[0], 16);
                    const uint32_t sl = lane / 3u;
                    if (lane < 9u && sl < rd.nsec) {
                        const uint32_t sec = sl == 0 ? rd.sec[0] : sl == 1 ? rd.sec[1] : rd.sec[2];
                        acc[(sec * kWarps + warp) * 3 + lane % 3u] += x;
                    }
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int k = 0; k < KA; ++k) {
            const uint32_t l = tid + uint32_t(k) * kT;
            if (l < amps) {
                const uint32_t x = xr | xl(k);
                psi[base + x] = sp[sw2(l)];
                if (BWD) lam[base + x] = sl[sw2(l)];
            }
        }
        __syncthreads();
    }
    if (BWD) {
        const uint32_t nv = sg.nsec * 3;
        for (uint32_t i = tid; i < nv; i += kT) {
            const uint32_t s2 = i / 3, c = i % 3;
            double sum = 0.0;
            for (int w = 0; w < kWarps; ++w) sum += acc[(s2 * kWarps + w) * 3 + c];
            kpart[size_t(blockIdx.x) * nv + i] = sum;
        }
        __threadfence();
        __syncthreads();
        __shared__ bool last;
        if (tid == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
        __syncthreads();
        if (last) { // fixed-order sum over CTAs
            __threadfence();
            for (uint32_t i = tid; i < nv; i += kT) {
                double sum = 0.0;
                for (uint32_t b = 0; b < gridDim.x; ++b) sum += __ldcg(kpart + size_t(b) * nv + i);
                K[size_t(sg.sec_begin) * 3 + i] = sum;
            }
            if (tid == 0) *ticket = 0;
        }
    }
}

} // namespace

C128Plan build_c128_plan(const qf_gate *gates, size_t n_gates, uint32_t n, uint64_t batch, int sms) {
    C128Plan P;
    for (size_t i = 0; i < n_gates; ++i) {
        const qf_gate &g = gates[i];
        if (g.kind == QF_GATE_ROTATION) {
            if (!P.ops.empty() && P.ops.back().type == 0 && P.ops.back().q == g.q0) {
                P.sec_cnt.back()++;
            } else {
                P.ops.push_back({0u, g.q0, uint32_t(P.sec_off.size()), 0u});
                P.sec_off.push_back(uint32_t(P.sec_gates.size()));
                P.sec_cnt.push_back(1u);
            }
            P.sec_gates.push_back(uint32_t(g.axis) | (g.param << 2));
        } else if (g.kind == QF_GATE_CZ) {
            if (P.ops.empty() || P.ops.back().type != 1)
                P.ops.push_back({1u, 0u, uint32_t(P.cz.size()), 0u});
            P.cz.push_back(g.q0 | (g.q1 << 8));
            P.ops.back().b++;
        } else {
            P.ops.push_back({2u, g.q1, g.q0, 0u});
        }
    }
    // op qubit (sections: the target; CNOT: the target) before the round fields reuse q
    std::vector<uint32_t> opq(P.ops.size());
    for (size_t i = 0; i < P.ops.size(); ++i) opq[i] = P.ops[i].q;
    // tile bits: kC128TileBits, or 10 when the batch gives fewer tiles than SMs
    // (measured at n = 12, batch 32: 0.84 ms at m = 10, 1.0 at m = 11, 1.55 at m = 8)
    uint32_t m = std::min<uint32_t>(n, kC128TileBits);
    if (m > 10 && (batch << (n - m)) < uint64_t(std::max(1, sms))) m = 10;
    const uint32_t nbase = std::min<uint32_t>(n, 3);
    const uint32_t R = std::min<uint32_t>(m, 3);
    size_t i = 0;
    uint32_t sec = 0;
    while (i < P.ops.size() || (P.ops.empty() && P.segs.empty())) {
        std::set<uint32_t> S;
        for (uint32_t q = 0; q < nbase; ++q) S.insert(q);
        uint32_t nsec = 0, ncp = 0, cz0 = 0;
        bool any_cz = false;
        size_t j = i;
        for (; j < P.ops.size(); ++j) {
            const C128Op &op = P.ops[j];
            const bool needs = op.type != 1;
            if (needs && !S.count(opq[j]) && S.size() + 1 > m) break;
            if (op.type == 0 && nsec == uint32_t(kC128MaxSec)) break;
            if (j - i == size_t(kC128MaxOps)) break;
            if (op.type == 1 && ncp + op.b > uint32_t(kC128MaxCzPairs)) break;
            if (needs) S.insert(opq[j]);
            if (op.type == 0) ++nsec;
            if (op.type == 1) {
                if (!any_cz) cz0 = op.a;
                any_cz = true;
                ncp += op.b;
            }
        }
        for (uint32_t q = 0; S.size() < m; ++q) S.insert(q);
        C128Seg sg{};
        sg.m = m;
        sg.nrest = n - m;
        sg.op_begin = uint32_t(i);
        sg.op_end = uint32_t(j);
        sg.sec_begin = sec;
        sg.nsec = nsec;
        sg.cz_begin = cz0; // the segment's CZ pairs are contiguous (appended in op order)
        sg.cz_count = ncp;
        for (int q = 0; q < 32; ++q) sg.lpos[q] = -1;
        uint32_t l = 0, r = 0;
        for (uint32_t q = 0; q < n; ++q) {
            if (S.count(q)) {
                sg.lq[l] = uint8_t(q);
                sg.lpos[q] = int8_t(l++);
            } else {
                sg.rq[r++] = uint8_t(q);
            }
        }
        // ---- rounds: up to kC128RoundSecs sections on at most R local bits plus the
        // CZ runs between them; a CNOT alone
        sg.round_begin = uint32_t(P.rounds.size());
        C128Round cur{};
        bool open = false;
        std::vector<uint32_t> cur_bits;
        auto close = [&] {
            if (!open) return;
            // pad the register bits to R, preferring pads that leave a conflict-free
            // quarter-warp (its three lowest thread bits distinct mod 3, sw2)
            std::vector<uint32_t> best;
            auto ok = [&](const std::vector<uint32_t> &bits) {
                std::vector<uint32_t> thr;
                for (uint32_t p = 0; p < m && thr.size() < 3; ++p)
                    if (std::find(bits.begin(), bits.end(), p) == bits.end()) thr.push_back(p);
                if (thr.size() < 3) return true;
                return (thr[0] % 3) != (thr[1] % 3) && (thr[0] % 3) != (thr[2] % 3) && (thr[1] % 3) != (thr[2] % 3);
            };
            std::vector<uint32_t> bits = cur_bits;
            std::function<bool(std::vector<uint32_t> &)> pad = [&](std::vector<uint32_t> &b) {
                if (b.size() == R) return ok(b);
                for (uint32_t p = 0; p < m; ++p) {
                    if (std::find(b.begin(), b.end(), p) != b.end()) continue;
                    b.push_back(p);
                    if (pad(b)) return true;
                    b.pop_back();
                }
                return false;
            };
            if (!pad(bits)) { // no conflict-free choice: lowest free positions
                bits = cur_bits;
                for (uint32_t p = 0; p < m && bits.size() < R; ++p)
                    if (std::find(bits.begin(), bits.end(), p) == bits.end()) bits.push_back(p);
            }
            std::sort(bits.begin(), bits.end());
            for (uint32_t k = 0; k < 4; ++k) {
                cur.bits[k] = k < bits.size() ? uint8_t(bits[k]) : 0;
                cur.gq[k] = k < bits.size() ? sg.lq[bits[k]] : 0;
            }
            for (uint32_t o = cur.op_begin; o < cur.op_end; ++o) {
                C128Op &op = P.ops[o];
                if (op.type == 0) {
                    const uint32_t p = uint32_t(sg.lpos[opq[o]]);
                    op.q = uint32_t(std::find(bits.begin(), bits.end(), p) - bits.begin());
                    cur.sbit[op.b] = uint8_t(op.q);
                } else if (op.type == 1) { // Q of every register offset j
                    uint32_t qo = 0;
                    for (uint32_t jo = 0; jo < (1u << R); ++jo) {
                        uint32_t par = 0;
                        for (uint32_t c = 0; c < op.b; ++c) {
                            const uint32_t pr = P.cz[op.a + c], a = pr & 255u, b = pr >> 8;
                            uint32_t ia = 4, ib = 4;
                            for (uint32_t k = 0; k < bits.size(); ++k) {
                                if (sg.lq[bits[k]] == a) ia = k;
                                if (sg.lq[bits[k]] == b) ib = k;
                            }
                            if (ia < 4 && ib < 4) par ^= ((jo >> ia) & (jo >> ib)) & 1u;
                        }
                        qo |= par << jo;
                    }
                    op.q = qo;
                }
            }
            P.rounds.push_back(cur);
            open = false;
        };
        for (size_t o = i; o < j; ++o) {
            const C128Op &op = P.ops[o];
            if (op.type == 2) {
                close();
                C128Round rd{};
                rd.kind = 1;
                rd.op_begin = uint32_t(o);
                rd.op_end = uint32_t(o + 1);
                P.rounds.push_back(rd);
                continue;
            }
            if (op.type == 0) {
                const uint32_t p = uint32_t(sg.lpos[opq[o]]);
                const bool have = std::find(cur_bits.begin(), cur_bits.end(), p) != cur_bits.end();
                // one section per register bit: the round applies all Rz(g) first and all
                // Rz(a) last (they commute with everything in the round but their own Ry)
                if (open && (cur.nsec == uint32_t(kC128RoundSecs) || have || cur_bits.size() == R)) close();
                if (!open) {
                    cur = C128Round{};
                    cur.op_begin = uint32_t(o);
                    cur_bits.clear();
                    open = true;
                }
                if (std::find(cur_bits.begin(), cur_bits.end(), p) == cur_bits.end()) cur_bits.push_back(p);
                P.ops[o].b = cur.nsec;                               // K slot
                cur.sec[cur.nsec++] = uint8_t(P.ops[o].a - sec);     // section within the segment
            } else {
                if (!open) {
                    cur = C128Round{};
                    cur.op_begin = uint32_t(o);
                    cur_bits.clear();
                    open = true;
                }
                cur.has_cz = 1;
            }
            cur.op_end = uint32_t(o + 1);
        }
        close();
        sg.round_end = uint32_t(P.rounds.size());
        if (sg.round_end - sg.round_begin > uint32_t(kC128MaxRounds))
            throw std::runtime_error("c128 plan: too many rounds in a segment");
        P.segs.push_back(sg);
        sec += nsec;
        if (j == i) break; // empty circuit: one segment that only copies
        i = j;
    }
    return P;
}

int c128_seg_grid(int sms, uint64_t tiles) {
    const uint64_t cap = uint64_t(sms) * 2; // 2 CTAs/SM (backward: 70 KiB smem, <= 128 registers)
    return int(std::max<uint64_t>(1, std::min(tiles, cap)));
}

cudaError_t launch_c128_prep(cudaStream_t st, int nsec, const uint32_t *off, const uint32_t *cnt,
                             const uint32_t *gates, const double *theta, double2 *secU) {
    if (nsec == 0) return cudaSuccess;
    c128_prep<<<(nsec + 127) / 128, 128, 0, st>>>(nsec, off, cnt, gates, theta, secU);
    return cudaGetLastError();
}

namespace {
std::atomic<uint64_t> g_c128_attr{0};
template <bool BWD, int R>
void launch_seg(cudaStream_t st, int grid, size_t smem, const C128Seg &sg, const C128Op *ops,
                const C128Round *rounds, const uint32_t *cz, const double2 *secU, double2 *psi,
                double2 *lam, int n, uint64_t tiles, double *kpart, unsigned *ticket, double *K) {
    seg_c128<BWD, R><<<grid, kT, smem, st>>>(sg, ops, rounds, cz, secU, psi, lam, n, tiles, kpart, ticket, K);
}
} // namespace

cudaError_t launch_c128_segment(cudaStream_t st, bool backward, int grid, const C128Seg &sg,
                                const C128Op *ops, const C128Round *rounds, const uint32_t *cz,
                                const double2 *secU, double2 *psi, double2 *lam, int n, uint32_t batch,
                                double *kpart, unsigned *ticket, double *K) {
    const uint64_t tiles = uint64_t(batch) << sg.nrest;
    const size_t amps = size_t(1) << sg.m;
    const size_t tabs = size_t(kC128MaxRounds) * (16 * sizeof(double2) + 4 * sizeof(double));
    const size_t smax = (size_t(2) << kC128TileBits) * sizeof(double2) + tabs +
                        size_t(kC128MaxSec) * kWarps * 3 * sizeof(double);
    const cudaError_t attr = once_per_device(g_c128_attr, [&] {
        cudaError_t e = cudaSuccess;
#define QF_C128_ATTR(B, R) \
        if (e == cudaSuccess) e = cudaFuncSetAttribute(seg_c128<B, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smax));
        QF_C128_ATTR(true, 1) QF_C128_ATTR(true, 2) QF_C128_ATTR(true, 3)
        QF_C128_ATTR(false, 1) QF_C128_ATTR(false, 2) QF_C128_ATTR(false, 3)
#undef QF_C128_ATTR
        return e;
    });
    if (attr != cudaSuccess) return attr;
    const int R = int(std::min<uint32_t>(sg.m, 3u));
    const size_t smem = amps * (backward ? 2 : 1) * sizeof(double2) + tabs +
                        (backward ? size_t(std::max<uint32_t>(sg.nsec, 1)) * kWarps * 3 * sizeof(double) : 0);
    if (backward) {
        if (R == 3) launch_seg<true, 3>(st, grid, smem, sg, ops, rounds, cz, secU, psi, lam, n, tiles, kpart, ticket, K);
        else if (R == 2) launch_seg<true, 2>(st, grid, smem, sg, ops, rounds, cz, secU, psi, lam, n, tiles, kpart, ticket, K);
        else launch_seg<true, 1>(st, grid, smem, sg, ops, rounds, cz, secU, psi, lam, n, tiles, kpart, ticket, K);
    } else {
        if (R == 3) launch_seg<false, 3>(st, grid, smem, sg, ops, rounds, cz, secU, psi, lam, n, tiles, kpart, ticket, K);
        else if (R == 2) launch_seg<false, 2>(st, grid, smem, sg, ops, rounds, cz, secU, psi, lam, n, tiles, kpart, ticket, K);
        else launch_seg<false, 1>(st, grid, smem, sg, ops, rounds, cz, secU, psi, lam, n, tiles, kpart, ticket, K);
    }
    return cudaGetLastError();
}

cudaError_t launch_c128_finalize(cudaStream_t st, int nsec, const uint32_t *off, const uint32_t *cnt,
                                 const uint32_t *gates, const double *theta, const double2 *secU,
                                 const double *K, double *grad) {
    if (nsec == 0) return cudaSuccess;
    c128_finalize<<<(nsec + 127) / 128, 128, 0, st>>>(nsec, off, cnt, gates, theta, secU, K, grad);
    return cudaGetLastError();
}

} // namespace qfb
