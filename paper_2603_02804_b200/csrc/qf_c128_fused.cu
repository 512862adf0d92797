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
// shared memory (m = min(n, 10); qubits 0..2 always local so every 8
// amplitudes are one 128-B line). One CTA loads a tile (psi, and lambda in
// the backward), runs the segment's ops on it between __syncthreads, and
// writes it back.
//
// Backward: for each section, in reverse, psi_in = U^dag psi_out and lam_in =
// U^dag lam_out (psi uncomputed in place: unitary in fp64, the same choice as
// the per-gate c128 path), and K = sum_pairs psi_in lam_in^dag (2x2) is
// accumulated. The gradient of rotation j of the section is
//   Re <lam_out| A_j dg_j B_j |psi_in> = Re Tr(M_j K),  M_j = B_j^dag g_j^dag dg_j B_j
// (B_j = the rotations before j, A_j after; rotation_derivative
// circuit.cpp:76-87), evaluated in fp64 by c128_finalize. K partials are
// reduced per warp (reduce-scatter), per CTA in fixed warp order, and over
// CTAs in fixed order by the last CTA of the segment: deterministic.
#include <algorithm>
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
    secU[4 * s + 0] = U.a;
    secU[4 * s + 1] = U.b;
    secU[4 * s + 2] = U.c;
    secU[4 * s + 3] = U.d;
}

// K layout per section: K00, K01, K10, K11 as (re, im) = 8 doubles.
__global__ void c128_finalize(int nsec, const uint32_t *off, const uint32_t *cnt,
                              const uint32_t *gates, const double *theta, const double *K,
                              double *grad) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nsec) return;
    const double *k = K + size_t(s) * 8;
    const Cx2 Kq = {make_double2(k[0], k[1]), make_double2(k[2], k[3]), make_double2(k[4], k[5]),
                    make_double2(k[6], k[7])};
    Cx2 B = ident();
    for (uint32_t i = 0; i < cnt[s]; ++i) {
        const uint32_t g = gates[off[s] + i];
        const int axis = int(g & 3u);
        double sn, cs;
        sincos(theta[g >> 2] / 2.0, &sn, &cs);
        const Cx2 u = rot(axis, cs, sn), du = rot(axis, -0.5 * sn, 0.5 * cs);
        const Cx2 M = mul(dag(B), mul(dag(u), mul(du, B)));
        const Cx2 MK = mul(M, Kq);
        grad[g >> 2] = MK.a.x + MK.d.x; // Re Tr(M K)
        B = mul(u, B);
    }
}

// Shared-memory slot of tile amplitude l: the low 3 bits are XORed with 7 when
// bit 3 is set, so the 8 lanes of a quarter-warp hit 8 distinct 16-B bank groups
// for pair accesses on every local bit (bits 0..2 would otherwise be 2-way
// conflicted) and for consecutive amplitudes.
__device__ __forceinline__ uint32_t sw(uint32_t l) { return l ^ (((l >> 3) & 1u) * 7u); }

__device__ __forceinline__ uint32_t insert0(uint32_t p, uint32_t pos) {
    return ((p >> pos) << (pos + 1)) | (p & ((1u << pos) - 1u));
}

__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gmem_src) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

struct U2 { // a section's unitary, or its adjoint
    double2 u00, u01, u10, u11;
};
__device__ __forceinline__ U2 load_u(const double2 *secU, uint32_t s, bool adjoint) {
    const double2 *u = secU + 4 * size_t(s);
    const double2 a = u[0], b = u[1], c = u[2], d = u[3];
    return adjoint ? U2{cj(a), cj(c), cj(b), cj(d)} : U2{a, b, c, d};
}
__device__ __forceinline__ void apply_u(const U2 &u, double2 &a, double2 &b) {
    const double2 a0 = a, b0 = b;
    a = cadd(cm(u.u00, a0), cm(u.u01, b0));
    b = cadd(cm(u.u10, a0), cm(u.u11, b0));
}
// K += [a; b] [la; lb]^dag (8 doubles: K00, K01, K10, K11 as re, im)
__device__ __forceinline__ void kacc(double (&k8)[8], double2 a, double2 b, double2 la, double2 lb) {
    const double2 k00 = cm(a, cj(la)), k01 = cm(a, cj(lb)), k10 = cm(b, cj(la)), k11 = cm(b, cj(lb));
    k8[0] += k00.x; k8[1] += k00.y; k8[2] += k01.x; k8[3] += k01.y;
    k8[4] += k10.x; k8[5] += k10.y; k8[6] += k11.x; k8[7] += k11.y;
}
// Warp sum of the 8 values (reduce-scatter over 8-lane groups, then across the
// groups), added by lanes 0..7 to this warp's accumulator slot.
__device__ __forceinline__ void kflush(double (&k8)[8], uint32_t lane, double *slot) {
#pragma unroll
    for (int m = 4; m >= 1; m >>= 1) {
        const bool up = (lane & uint32_t(m)) != 0;
#pragma unroll
        for (int i = 0; i < m; ++i) {
            const double send = up ? k8[i] : k8[i + m];
            const double keep = up ? k8[i + m] : k8[i];
            k8[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
        }
    }
    double v = k8[0];
    v += __shfl_xor_sync(0xffffffffu, v, 8);
    v += __shfl_xor_sync(0xffffffffu, v, 16);
    if (lane < 8) slot[lane] += v;
}

template <bool BWD>
__global__ void __launch_bounds__(kT, 2) seg_c128(const C128Seg sg, const C128Op *__restrict__ ops,
                                               const uint32_t *__restrict__ czp,
                                               const double2 *__restrict__ secU, double2 *psi,
                                               double2 *lam, int n, uint64_t tiles, double *kpart,
                                               unsigned *ticket, double *K) {
    extern __shared__ double2 sm[];
    const uint32_t amps = 1u << sg.m, pairs = amps >> 1;
    constexpr uint32_t kBufs = BWD ? 2u : 1u; // psi (+ lambda) per tile buffer
    // two tile buffers: tile i+1 is copied in (cp.async) while tile i is processed
    double *acc = reinterpret_cast<double *>(sm + 2 * kBufs * amps); // [sec][warp][8]
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
    // the segment's qubit maps, indexed at run time: shared copies (not a local
    // copy of the parameter block)
    __shared__ int8_t lpos[32];
    __shared__ uint8_t lq[16], rq[32];
    if (tid == 0) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            lpos[i] = sg.lpos[i];
            rq[i] = sg.rq[i];
            if (i < 16) lq[i] = sg.lq[i];
        }
    }
    // the segment's ops, section unitaries and CZ pairs, staged once per CTA
    __shared__ C128Op ops_s[kC128MaxOps];
    __shared__ double2 u_s[kC128MaxSec * 4];
    __shared__ uint32_t cz_s[kC128MaxCzPairs];
    const uint32_t nops = sg.op_end - sg.op_begin;
    for (uint32_t i = tid; i < nops; i += kT) ops_s[i] = ops[sg.op_begin + i];
    for (uint32_t i = tid; i < sg.nsec * 4; i += kT) u_s[i] = secU[size_t(sg.sec_begin) * 4 + i];
    for (uint32_t i = tid; i < sg.cz_count; i += kT) cz_s[i] = czp[sg.cz_begin + i];
    if (BWD)
        for (uint32_t i = tid; i < sg.nsec * 64; i += kT) acc[i] = 0.0;
    __syncthreads();
    constexpr int KA = (1 << kC128TileBits) / kT; // amplitudes per thread
    // local part of the global index of this thread's amplitudes (fixed per segment)
    uint32_t xl[KA];
#pragma unroll
    for (int k = 0; k < KA; ++k) {
        const uint32_t l = tid + uint32_t(k) * kT;
        uint32_t x = 0;
        for (uint32_t j = 0; j < sg.m; ++j) x |= ((l >> j) & 1u) << lq[j];
        xl[k] = x;
    }
    // Q(xl) of every CZ run of the segment (op.q = its index < kC128MaxCz)
    uint32_t qlb[KA];
#pragma unroll
    for (int k = 0; k < KA; ++k) qlb[k] = 0;
    for (uint32_t i = 0; i < nops; ++i) {
        const C128Op op = ops_s[i];
        if (op.type != 1) continue;
#pragma unroll
        for (int k = 0; k < KA; ++k) {
            uint32_t f = 0;
            for (uint32_t c = 0; c < op.b; ++c) {
                const uint32_t w = cz_s[op.a - sg.cz_begin + c];
                f ^= (xl[k] >> (w & 255u)) & (xl[k] >> (w >> 8)) & 1u;
            }
            qlb[k] |= f << op.q;
        }
    }
    auto tile_xr = [&](uint64_t t) {
        const uint32_t r = uint32_t(t) & ((1u << sg.nrest) - 1u);
        uint32_t xr = 0;
        for (uint32_t k = 0; k < sg.nrest; ++k) xr |= ((r >> k) & 1u) << rq[k];
        return xr;
    };
    auto fetch = [&](uint64_t t, uint32_t buf) {
        const uint64_t base = (t >> sg.nrest) << n;
        const uint32_t xr = tile_xr(t);
        double2 *dp = sm + buf * kBufs * amps;
#pragma unroll
        for (int k = 0; k < KA; ++k) {
            const uint32_t l = tid + uint32_t(k) * kT;
            if (l < amps) {
                cp_async16(dp + sw(l), psi + base + (xr | xl[k]));
                if (BWD) cp_async16(dp + amps + sw(l), lam + base + (xr | xl[k]));
            }
        }
        cp_async_commit();
    };
    uint32_t it = 0;
    if (blockIdx.x < tiles) fetch(blockIdx.x, 0);
    for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
        const uint32_t buf = it & 1u;
        double2 *sp = sm + buf * kBufs * amps, *sl = sp + amps;
        const uint64_t base = (t >> sg.nrest) << n;
        const uint32_t xr_cur = tile_xr(t);
        uint32_t xs[KA];
#pragma unroll
        for (int k = 0; k < KA; ++k) xs[k] = xr_cur | xl[k];
        cp_async_wait_all();
        __syncthreads();
        if (t + gridDim.x < tiles) fetch(t + gridDim.x, buf ^ 1u);
        for (uint32_t ii = 0; ii < nops; ++ii) {
            const C128Op op = ops_s[BWD ? nops - 1 - ii : ii];
            if (op.type == 0 && ii + 1 < nops && amps >= 4) {
                const C128Op op2 = ops_s[BWD ? nops - 2 - ii : ii + 1];
                if (op2.type == 0 && op2.q != op.q) {
                    // two sections on different qubits in one round: each thread
                    // owns a quad (bits p1, p2) and applies (or undoes) op then op2
                    // in registers; K of both is measured after both are undone
                    // (K of a qubit is invariant under gates on other qubits)
                    const uint32_t p1 = uint32_t(lpos[op.q]), p2 = uint32_t(lpos[op2.q]);
                    const uint32_t lo = min(p1, p2), hi = max(p1, p2);
                    const U2 ua = load_u(u_s, op.a - sg.sec_begin, BWD), ub = load_u(u_s, op2.a - sg.sec_begin, BWD);
                    double ka[8] = {0, 0, 0, 0, 0, 0, 0, 0}, kb[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                    if (tid < (amps >> 2)) { // amps / 4 <= kT: one quad per thread
                        const uint32_t b0 = insert0(insert0(tid, lo), hi);
                        uint32_t ix[2][2];
                        double2 v[2][2], w[2][2];
#pragma unroll
                        for (int i = 0; i < 2; ++i)
#pragma unroll
                            for (int j = 0; j < 2; ++j) {
                                ix[i][j] = sw(b0 | (uint32_t(i) << p1) | (uint32_t(j) << p2));
                                v[i][j] = sp[ix[i][j]];
                                if (BWD) w[i][j] = sl[ix[i][j]];
                            }
#pragma unroll
                        for (int j = 0; j < 2; ++j) {
                            apply_u(ua, v[0][j], v[1][j]);
                            if (BWD) apply_u(ua, w[0][j], w[1][j]);
                        }
#pragma unroll
                        for (int i = 0; i < 2; ++i) {
                            apply_u(ub, v[i][0], v[i][1]);
                            if (BWD) apply_u(ub, w[i][0], w[i][1]);
                        }
                        if (BWD) {
#pragma unroll
                            for (int j = 0; j < 2; ++j) kacc(ka, v[0][j], v[1][j], w[0][j], w[1][j]);
#pragma unroll
                            for (int i = 0; i < 2; ++i) kacc(kb, v[i][0], v[i][1], w[i][0], w[i][1]);
                        }
#pragma unroll
                        for (int i = 0; i < 2; ++i)
#pragma unroll
                            for (int j = 0; j < 2; ++j) {
                                sp[ix[i][j]] = v[i][j];
                                if (BWD) sl[ix[i][j]] = w[i][j];
                            }
                    }
                    if (BWD) {
                        kflush(ka, lane, acc + ((op.a - sg.sec_begin) * 8 + warp) * 8);
                        kflush(kb, lane, acc + ((op2.a - sg.sec_begin) * 8 + warp) * 8);
                    }
                    ++ii;
                    __syncthreads();
                    continue;
                }
            }
            if (op.type == 0) { // a single section
                const uint32_t pos = uint32_t(lpos[op.q]);
                const U2 u = load_u(u_s, op.a - sg.sec_begin, BWD);
                double k8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                for (uint32_t p = tid; p < pairs; p += kT) {
                    const uint32_t i0 = sw(insert0(p, pos)), i1 = sw(insert0(p, pos) | (1u << pos));
                    double2 a = sp[i0], b = sp[i1];
                    apply_u(u, a, b);
                    sp[i0] = a;
                    sp[i1] = b;
                    if (BWD) {
                        double2 la = sl[i0], lb = sl[i1];
                        apply_u(u, la, lb);
                        sl[i0] = la;
                        sl[i1] = lb;
                        kacc(k8, a, b, la, lb);
                    }
                }
                if (BWD) kflush(k8, lane, acc + ((op.a - sg.sec_begin) * 8 + warp) * 8);
            } else if (op.type == 1) { // CZ run: one sign per amplitude
                // Q(xr | xl) = Q(xr) ^ Q(xl) ^ parity(xl & M(xr)), M(xr) = the qubits
                // with an odd number of CZ partners set in xr: the per-pair loop runs
                // once per tile (warp-uniform) instead of once per amplitude, and
                // Q(xl) of this thread's amplitudes is precomputed (qlb, bit op.q).
                uint32_t qr = 0, M = 0;
                for (uint32_t c = 0; c < op.b; ++c) {
                    const uint32_t w = cz_s[op.a - sg.cz_begin + c], a = w & 255u, b = w >> 8;
                    const uint32_t ra = (xr_cur >> a) & 1u, rb = (xr_cur >> b) & 1u;
                    qr ^= ra & rb;
                    M ^= (ra << b) ^ (rb << a);
                }
#pragma unroll
                for (int k = 0; k < KA; ++k) {
                    const uint32_t l = tid + uint32_t(k) * kT;
                    if (l < amps && (qr ^ ((qlb[k] >> op.q) & 1u) ^ (__popc(xl[k] & M) & 1u))) {
                        sp[sw(l)] = make_double2(-sp[sw(l)].x, -sp[sw(l)].y);
                        if (BWD) sl[sw(l)] = make_double2(-sl[sw(l)].x, -sl[sw(l)].y);
                    }
                }
            } else { // CNOT(control a, target q): self-inverse
                const uint32_t pos = uint32_t(lpos[op.q]);
                const int cpos = lpos[op.a];
                for (uint32_t p = tid; p < pairs; p += kT) {
                    const uint32_t i0 = insert0(p, pos), i1 = i0 | (1u << pos);
                    const uint32_t ctl = cpos >= 0 ? (i0 >> cpos) & 1u : (xr_cur >> op.a) & 1u;
                    if (ctl) {
                        double2 tmp = sp[sw(i0)];
                        sp[sw(i0)] = sp[sw(i1)];
                        sp[sw(i1)] = tmp;
                        if (BWD) {
                            tmp = sl[sw(i0)];
                            sl[sw(i0)] = sl[sw(i1)];
                            sl[sw(i1)] = tmp;
                        }
                    }
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int k = 0; k < KA; ++k) {
            const uint32_t l = tid + uint32_t(k) * kT;
            if (l < amps) {
                psi[base + xs[k]] = sp[sw(l)];
                if (BWD) lam[base + xs[k]] = sl[sw(l)];
            }
        }
        __syncthreads();
    }
    if (BWD) {
        const uint32_t nv = sg.nsec * 8;
        for (uint32_t i = tid; i < nv; i += kT) {
            const uint32_t s = i >> 3, c = i & 7u;
            double sum = 0.0;
            for (int w = 0; w < kT / 32; ++w) sum += acc[(s * 8 + w) * 8 + c];
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
                K[size_t(sg.sec_begin) * 8 + i] = sum;
            }
            if (tid == 0) *ticket = 0;
        }
    }
}

} // namespace

C128Plan build_c128_plan(const qf_gate *gates, size_t n_gates, uint32_t n) {
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
    const uint32_t m = std::min<uint32_t>(n, kC128TileBits);
    const uint32_t nbase = std::min<uint32_t>(n, 3);
    size_t i = 0;
    uint32_t sec = 0;
    while (i < P.ops.size() || (P.ops.empty() && P.segs.empty())) {
        std::set<uint32_t> S;
        for (uint32_t q = 0; q < nbase; ++q) S.insert(q);
        uint32_t nsec = 0, ncz = 0, ncp = 0, cz0 = 0;
        size_t j = i;
        for (; j < P.ops.size(); ++j) {
            const C128Op &op = P.ops[j];
            const bool needs = op.type != 1;
            if (needs && !S.count(op.q) && S.size() + 1 > m) break;
            if (op.type == 0 && nsec == uint32_t(kC128MaxSec)) break;
            if (op.type == 1 && ncz == uint32_t(kC128MaxCz)) break;
            if (j - i == size_t(kC128MaxOps)) break;
            if (op.type == 1 && ncp + op.b > uint32_t(kC128MaxCzPairs)) break;
            if (needs) S.insert(op.q);
            if (op.type == 0) ++nsec;
            if (op.type == 1) {
                if (ncz == 0) cz0 = op.a;
                P.ops[j].q = ncz++; // index of the CZ run within its segment
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
        P.segs.push_back(sg);
        sec += nsec;
        if (j == i) break; // empty circuit: one segment that only copies
        i = j;
    }
    return P;
}

int c128_seg_grid(int sms, uint64_t tiles) {
    const uint64_t cap = uint64_t(sms) * 2; // 2 CTAs/SM (backward: 80 KiB smem, <= 128 registers)
    return int(std::max<uint64_t>(1, std::min(tiles, cap)));
}

cudaError_t launch_c128_prep(cudaStream_t st, int nsec, const uint32_t *off, const uint32_t *cnt,
                             const uint32_t *gates, const double *theta, double2 *secU) {
    if (nsec == 0) return cudaSuccess;
    c128_prep<<<(nsec + 127) / 128, 128, 0, st>>>(nsec, off, cnt, gates, theta, secU);
    return cudaGetLastError();
}

cudaError_t launch_c128_segment(cudaStream_t st, bool backward, int grid, const C128Seg &sg,
                                const C128Op *ops, const uint32_t *cz, const double2 *secU,
                                double2 *psi, double2 *lam, int n, uint32_t batch, double *kpart,
                                unsigned *ticket, double *K) {
    const uint64_t tiles = uint64_t(batch) << sg.nrest;
    const size_t amps = size_t(1) << sg.m;
    if (backward) {
        const size_t smem = amps * 4 * sizeof(double2) + size_t(kC128MaxSec) * 64 * sizeof(double);
        static std::atomic<uint64_t> done{0};
        const cudaError_t attr = once_per_device(done, [] {
            return cudaFuncSetAttribute(
                seg_c128<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                int((size_t(4) << kC128TileBits) * sizeof(double2) + size_t(kC128MaxSec) * 64 * sizeof(double)));
        });
        if (attr != cudaSuccess) return attr;
        seg_c128<true><<<grid, kT, smem, st>>>(sg, ops, cz, secU, psi, lam, n, tiles, kpart, ticket, K);
    } else {
        const size_t smem = amps * 2 * sizeof(double2);
        seg_c128<false><<<grid, kT, smem, st>>>(sg, ops, cz, secU, psi, lam, n, tiles, kpart, ticket, K);
    }
    return cudaGetLastError();
}

cudaError_t launch_c128_finalize(cudaStream_t st, int nsec, const uint32_t *off, const uint32_t *cnt,
                                 const uint32_t *gates, const double *theta, const double *K,
                                 double *grad) {
    if (nsec == 0) return cudaSuccess;
    c128_finalize<<<(nsec + 127) / 128, 128, 0, st>>>(nsec, off, cnt, gates, theta, K, grad);
    return cudaGetLastError();
}

} // namespace qfb
