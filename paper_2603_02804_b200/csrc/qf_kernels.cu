// sm_100a kernels of the fused forward / adjoint-gradient path.
//
// Device model. Every single-qubit run of the circuit is
// written U = e^{i delta} Rz(alpha) Ry(beta) Rz(gamma); the Rz factors and all
// CZ gates are diagonal, so each device *stage* s is
//     psi <- Ry_stage(s) * D_s * psi,     D_s(x) = (-1)^{Q_s(x)} e^{i sum_q w_sq x_q},
// and the circuit is stages 0..S-1 followed by a final diagonal D_f that the
// observable step folds into O' = D_f^dag O D_f. A stage moves the batch
// store through HBM once per *pass*: pass A keeps qubits 0..11 resident in a
// 4096-amplitude shared-memory tile, pass B keeps qubits 0..3 plus the top
// eight (n <= 20). The adjoint backward undoes the stage on psi and lambda in
// the same tiles and accumulates, per (stage, qubit), the 2x2 cross
// correlation K = sum psi lambda^dag at the point just before Ry(beta); the
// parameter gradients of the reference's Rx/Ry/Rz gates follow exactly from K
// on the host-independent finalize kernel (finalize_kernel).
//
// Reference semantics restated (paths under /root/reference/proj):
//   forward of a fused op            engine.cpp:61-109, :111-136, :638-658
//   expectation / adjoint seed       engine.cpp:346-435
//   block backward (grad = Re<lam|du|psi_in>)  engine.cpp:265-342
//   gradient driver                  engine.cpp:716-755
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "qf_internal.h"

namespace qfb {
namespace {

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
__device__ __forceinline__ void tma_load5(void *dst, const CUtensorMap *map, uint64_t *bar,
                                          int c0, int c1, int c2, int c3, int c4) {
    asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(dst)),
                 "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
                 "r"(c4), "r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void tma_store5(const CUtensorMap *map, const void *src, int c0,
                                           int c1, int c2, int c3, int c4) {
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group"
                 " [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(su32(src))
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

// ------------------------------------------------------- tile addressing
// Byte offset of register j (0..15) of thread tau (0..255) in group phase G.
// Group G holds local bits [4G, 4G+4) in registers. The tile is 256 rows of
// 128 B with the TMA 128B swizzle: 16-B chunk c of row r sits at c ^ (r & 7).
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
// Local (12-bit) index of register j of thread tau in group G.
template <int G> __device__ __forceinline__ uint32_t gloc(uint32_t tau, int j) {
    if (G == 0) return (tau << 4) | uint32_t(j);
    if (G == 1) return (tau & 15u) | (uint32_t(j) << 4) | ((tau >> 4) << 8);
    return tau | (uint32_t(j) << 8);
}
__device__ __forceinline__ uint32_t swz(uint32_t l) {
    const uint32_t r = l >> 4, c = l & 15u;
    return (r << 7) | ((((c >> 1) ^ r) & 7u) << 4) | ((c & 1u) << 3);
}

template <int G>
__device__ __forceinline__ void lds16(const uint8_t *tile, uint32_t tau, float2 (&v)[16]) {
    if (G == 0) {
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
            const float4 t = *reinterpret_cast<const float4 *>(tile + goff<0>(tau, j));
            v[j] = make_float2(t.x, t.y);
            v[j + 1] = make_float2(t.z, t.w);
        }
    } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = *reinterpret_cast<const float2 *>(tile + goff<G>(tau, j));
    }
}
template <int G>
__device__ __forceinline__ void sts16(uint8_t *tile, uint32_t tau, const float2 (&v)[16]) {
    if (G == 0) {
#pragma unroll
        for (int j = 0; j < 16; j += 2)
            *reinterpret_cast<float4 *>(tile + goff<0>(tau, j)) =
                make_float4(v[j].x, v[j].y, v[j + 1].x, v[j + 1].y);
    } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) *reinterpret_cast<float2 *>(tile + goff<G>(tau, j)) = v[j];
    }
}

// --------------------------------------------------------- gate algebra
// Ry(beta) = [[c, -s], [s, c]] (circuit.cpp:67-68) on register bit B.
template <int B> __device__ __forceinline__ void ry_fwd(float2 (&v)[16], float c, float s) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        if (j & (1 << B)) continue;
        const float2 a = v[j], b = v[j | (1 << B)];
        v[j] = make_float2(c * a.x - s * b.x, c * a.y - s * b.y);
        v[j | (1 << B)] = make_float2(s * a.x + c * b.x, s * a.y + c * b.y);
    }
}
template <int B> __device__ __forceinline__ void ry_bwd(float2 (&v)[16], float c, float s) {
    ry_fwd<B>(v, c, -s);
}
// K_ab += psi_a conj(lam_b) over the pairs of register bit B. k[0..7] =
// (K00, K01, K10, K11) as (re, im).
template <int B>
__device__ __forceinline__ void kacc(const float2 (&p)[16], const float2 (&l)[16], float *k) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        if (j & (1 << B)) continue;
        const float2 p0 = p[j], p1 = p[j | (1 << B)], l0 = l[j], l1 = l[j | (1 << B)];
        k[0] += p0.x * l0.x + p0.y * l0.y;
        k[1] += p0.y * l0.x - p0.x * l0.y;
        k[2] += p0.x * l1.x + p0.y * l1.y;
        k[3] += p0.y * l1.x - p0.x * l1.y;
        k[4] += p1.x * l0.x + p1.y * l0.y;
        k[5] += p1.y * l0.x - p1.x * l0.y;
        k[6] += p1.x * l1.x + p1.y * l1.y;
        k[7] += p1.y * l1.x - p1.x * l1.y;
    }
}
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) { // conj(a) * b
    return make_float2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}

// Reduce-scatter of 32 per-lane values across the warp: afterwards lane L
// holds the warp sum of value L (31 shuffles instead of 160).
__device__ __forceinline__ float warp_reduce_scatter32(float (&v)[32]) {
    const uint32_t lane = threadIdx.x & 31u;
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        const bool up = (lane & m) != 0;
#pragma unroll
        for (int i = 0; i < m; ++i) {
            const float send = up ? v[i] : v[i + m];
            const float keep = up ? v[i + m] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
        }
    }
    return v[0];
}

// Parity of the CZ quadratic form restricted to a bit set v.
__device__ __forceinline__ uint32_t qform(const CzSet *cz, uint32_t v) {
    uint32_t par = 0, w = v;
    while (w) {
        const int q = __ffs(w) - 1;
        w &= w - 1;
        par ^= __popc(v & cz->adjlo[q]);
    }
    return par & 1u;
}
// 16-bit mask m with bit j = parity(j & M) for a 4-bit M.
__device__ __forceinline__ uint32_t linmask4(uint32_t M) {
    uint32_t m = 0;
    if (M & 1u) m ^= 0xAAAAu;
    if (M & 2u) m ^= 0xCCCCu;
    if (M & 4u) m ^= 0xF0F0u;
    if (M & 8u) m ^= 0xFF00u;
    return m;
}

// Diagonal D_s in pass-A layout for one thread in group 0 (row = tau).
struct DiagCtx {
    float2 base;     // e^{i phi(tile, row)}
    uint32_t sgn;    // bit j: sign of register j
};
__device__ __forceinline__ DiagCtx diag_ctx(uint32_t tau, uint32_t tilebits /* qubits >= 12 */,
                                            const float2 *trow, const float2 *tt1,
                                            const float2 *tt2, const CzSet *cz) {
    DiagCtx d;
    float2 b = trow[tau];
    if (tilebits) {
        b = cmul(b, cmul(tt1[tilebits & 255u], tt2[(tilebits >> 8) & 255u]));
    }
    d.base = b;
    d.sgn = 0;
    if (cz) {
        const uint32_t hi = tilebits << 12;
        uint32_t qt = qform(cz, hi), mt = 0, rt = 0;
        uint32_t w = hi;
        while (w) {
            const int q = __ffs(w) - 1;
            w &= w - 1;
            mt ^= cz->adj[q] & 15u;
            rt ^= (cz->adj[q] >> 4) & 255u;
        }
        const uint32_t ri = cz->rowinfo[tau];
        const uint32_t sbase = (qt ^ (ri >> 4) ^ __popc(tau & rt)) & 1u;
        d.sgn = (sbase ? 0xFFFFu : 0u) ^ cz->qcol ^ linmask4(mt ^ (ri & 15u));
    }
    return d;
}
template <bool CONJ>
__device__ __forceinline__ void apply_diag(float2 (&v)[16], const DiagCtx &d,
                                           const float2 *tcol_s) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        float2 g = cmul(d.base, tcol_s[j]);
        const uint32_t flip = (d.sgn << (31 - j)) & 0x80000000u;
        g.x = __uint_as_float(__float_as_uint(g.x) ^ flip);
        g.y = __uint_as_float(__float_as_uint(g.y) ^ flip);
        v[j] = CONJ ? cmulc(g, v[j]) : cmul(g, v[j]);
    }
}

// ---------------------------------------------------------- group phases
// Forward: (D_s on group 0) then Ry on every rotated bit of the group.
template <int G>
__device__ __forceinline__ void phase_fwd(uint8_t *tile, uint32_t tau, uint32_t rot,
                                          const float2 *ry_s, bool diag, const DiagCtx &d,
                                          const float2 *tcol_s) {
    float2 v[16];
    lds16<G>(tile, tau, v);
    if (G == 0 && diag) apply_diag<false>(v, d, tcol_s);
    if (rot & (1u << (4 * G + 0))) ry_fwd<0>(v, ry_s[4 * G + 0].x, ry_s[4 * G + 0].y);
    if (rot & (1u << (4 * G + 1))) ry_fwd<1>(v, ry_s[4 * G + 1].x, ry_s[4 * G + 1].y);
    if (rot & (1u << (4 * G + 2))) ry_fwd<2>(v, ry_s[4 * G + 2].x, ry_s[4 * G + 2].y);
    if (rot & (1u << (4 * G + 3))) ry_fwd<3>(v, ry_s[4 * G + 3].x, ry_s[4 * G + 3].y);
    sts16<G>(tile, tau, v);
}

// Backward: undo Ry on psi and lambda, accumulate K for the bit, then (group
// 0) undo D_s. The warp's K partials land in acc[warp][4G + b][8] (fp64).
template <int G>
__device__ __forceinline__ void phase_bwd(uint8_t *pt, uint8_t *lt, uint32_t tau, uint32_t rot,
                                          uint32_t meas, const float2 *ry_s, bool diag,
                                          const DiagCtx &d, const float2 *tcol_s,
                                          double *acc_w) {
    float2 p[16], l[16];
    lds16<G>(pt, tau, p);
    lds16<G>(lt, tau, l);
    float k[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) k[i] = 0.f;
#define QF_BWD_BIT(B)                                                                     \
    if (rot & (1u << (4 * G + B))) {                                                      \
        const float c = ry_s[4 * G + B].x, s = ry_s[4 * G + B].y;                         \
        ry_bwd<B>(p, c, s);                                                               \
        ry_bwd<B>(l, c, s);                                                               \
    }                                                                                     \
    if (meas & (1u << (4 * G + B))) kacc<B>(p, l, k + 8 * B);
    QF_BWD_BIT(0)
    QF_BWD_BIT(1)
    QF_BWD_BIT(2)
    QF_BWD_BIT(3)
#undef QF_BWD_BIT
    if (G == 0 && diag) {
        apply_diag<true>(p, d, tcol_s);
        apply_diag<true>(l, d, tcol_s);
    }
    sts16<G>(pt, tau, p);
    sts16<G>(lt, tau, l);
    if (meas & (0xFu << (4 * G))) {
        const float r = warp_reduce_scatter32(k);
        const uint32_t lane = threadIdx.x & 31u;
        acc_w[(4 * G + (lane >> 3)) * 8 + (lane & 7u)] += static_cast<double>(r);
    }
}

// ------------------------------------------------------ streaming pass
constexpr int kMaxDynSmem = 227 * 1024;

struct PassSmem {
    // tiles first (1024-aligned), then the small stuff
    static constexpr size_t tiles(bool bwd) { return size_t(2) * kTileBytes * (bwd ? 2 : 1); }
    static constexpr size_t bytes(bool bwd) {
        return tiles(bwd) + 64 /*mbar*/ + 12 * 8 /*ry*/ + 16 * 8 /*tcol*/ + 32 /*pad*/ +
               (bwd ? 8 * 12 * 8 * 8 : 0) + 1024 /*align*/;
    }
};

__device__ __forceinline__ uint8_t *align1024(uint8_t *p) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    return reinterpret_cast<uint8_t *>((a + 1023) & ~uintptr_t(1023));
}

template <bool BWD>
__global__ void __launch_bounds__(kThreads, BWD ? 1 : 2)
    pass_kernel(const __grid_constant__ PassParams p, const __grid_constant__ CUtensorMap m_in,
                const __grid_constant__ CUtensorMap m_out,
                const __grid_constant__ CUtensorMap m_lam) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    constexpr size_t kBuf = size_t(kTileBytes) * (BWD ? 2 : 1);
    uint8_t *buf[2] = {smem, smem + kBuf};
    uint8_t *tail = smem + 2 * kBuf;
    uint64_t *mbar = reinterpret_cast<uint64_t *>(tail);
    float2 *ry_s = reinterpret_cast<float2 *>(tail + 64);
    float2 *tcol_s = ry_s + 12;
    double *acc = reinterpret_cast<double *>(tail + 64 + 12 * 8 + 16 * 8 + 32);
    const uint32_t tid = threadIdx.x, warp = tid >> 5;

    if (tid < 12) {
        const int q = p.qmap[tid];
        ry_s[tid] = (p.rot_mask >> tid) & 1u ? p.ry[q] : make_float2(1.f, 0.f);
    }
    if (tid < 16) tcol_s[tid] = p.has_diag ? p.tcol[tid] : make_float2(1.f, 0.f);
    if (BWD) {
        for (int i = tid; i < 8 * 12 * 8; i += kThreads) acc[i] = 0.0;
    }
    if (tid == 0) {
        prefetch_map(&m_in);
        prefetch_map(&m_out);
        if (BWD) prefetch_map(&m_lam);
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const int lo_mask = (1 << p.tile_lo_bits) - 1, hi_mask = (1 << p.tile_hi_bits) - 1;
    const int sample_shift = p.tile_lo_bits + p.tile_hi_bits;
    auto issue_load = [&](int t, int b) {
        const int c1 = t & lo_mask, c3 = (t >> p.tile_lo_bits) & hi_mask, c4 = t >> sample_shift;
        mbar_expect_tx(&mbar[b], uint32_t(kBuf));
        tma_load5(buf[b], &m_in, &mbar[b], 0, c1, 0, c3, c4);
        if (BWD) tma_load5(buf[b] + kTileBytes, &m_lam, &mbar[b], 0, c1, 0, c3, c4);
    };
    const int stride = gridDim.x;
    if (tid == 0) {
        if ((int)blockIdx.x < p.tiles) issue_load(blockIdx.x, 0);
        if ((int)blockIdx.x + stride < p.tiles) issue_load(blockIdx.x + stride, 1);
    }
    const bool diag = p.has_diag != 0;
    const uint32_t rot = p.rot_mask, meas = p.meas_mask;
    int it = 0;
    for (int t = blockIdx.x; t < p.tiles; t += stride, ++it) {
        const int b = it & 1;
        mbar_wait(&mbar[b], (it >> 1) & 1);
        uint8_t *pt = buf[b];
        DiagCtx d{};
        if (diag) {
            const uint32_t tilebits = uint32_t((t >> p.tile_lo_bits) & hi_mask); // pass A: qubits 12..
            d = diag_ctx(tid, tilebits, p.trow, p.tt1, p.tt2, p.cz);
        }
        if (!BWD) {
            if (diag || (rot & 0xFu)) {
                phase_fwd<0>(pt, tid, rot, ry_s, diag, d, tcol_s);
                __syncthreads();
            }
            if (rot & 0xF0u) {
                phase_fwd<1>(pt, tid, rot, ry_s, false, d, tcol_s);
                __syncthreads();
            }
            if (rot & 0xF00u) {
                phase_fwd<2>(pt, tid, rot, ry_s, false, d, tcol_s);
            }
        } else {
            uint8_t *lt = pt + kTileBytes;
            double *acc_w = acc + warp * 12 * 8;
            if (rot & 0xF00u) {
                phase_bwd<2>(pt, lt, tid, rot, meas, ry_s, false, d, tcol_s, acc_w);
                __syncthreads();
            }
            if (rot & 0xF0u) {
                phase_bwd<1>(pt, lt, tid, rot, meas, ry_s, false, d, tcol_s, acc_w);
                __syncthreads();
            }
            if (diag || (rot & 0xFu)) {
                phase_bwd<0>(pt, lt, tid, rot, meas, ry_s, diag, d, tcol_s, acc_w);
            }
        }
        fence_async_smem();
        __syncthreads();
        if (tid == 0) {
            const int c1 = t & lo_mask, c3 = (t >> p.tile_lo_bits) & hi_mask, c4 = t >> sample_shift;
            if (!BWD || p.write_psi) tma_store5(&m_out, pt, 0, c1, 0, c3, c4);
            if (BWD) tma_store5(&m_lam, pt + kTileBytes, 0, c1, 0, c3, c4);
            bulk_commit();
            const int tn = t + 2 * stride;
            if (tn < p.tiles) {
                bulk_wait_read0();
                issue_load(tn, b);
            }
        }
    }
    if (tid == 0) bulk_wait0();
    if (BWD) {
        __syncthreads();
        if (tid < 96) {
            const int lb = tid >> 3, c = tid & 7;
            if ((meas >> lb) & 1u) {
                double s = 0.0;
#pragma unroll
                for (int w = 0; w < 8; ++w) s += acc[(w * 12 + lb) * 8 + c];
                p.kpart[size_t(blockIdx.x) * size_t(p.kstride) + size_t(p.qmap[lb]) * 8 + c] = s;
            }
        }
    }
}

// ------------------------------------------------------ observable step
// 2 * phase_O(t) * D_f(t) * conj(D_f(x)) with t = x ^ X: the adjoint seed
// lambda = 2 O' psi of the folded observable O' = D_f^dag O D_f
// (seed_adjoint_kernel engine.cpp:411-435 and pauli_phase engine.cpp:346-372).
__device__ __forceinline__ float2 seed_factor(uint32_t x, uint64_t X, uint64_t Z, uint32_t y,
                                              const double *wf, const CzSet *czf) {
    const uint32_t t = x ^ uint32_t(X);
    double ang = 0.0;
    uint32_t xm = uint32_t(X);
    while (xm) {
        const int q = __ffs(xm) - 1;
        xm &= xm - 1;
        ang += ((x >> q) & 1u) ? -wf[q] : wf[q];
    }
    uint32_t par = __popc(t & uint32_t(Z));
    if (czf) par += qform(czf, x) ^ qform(czf, t);
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

// Streaming observable step (n > 12): lambda = 2 O' psi and per-chunk fp64
// partials of E_s = <psi|O'|psi> (expectation_kernel engine.cpp:374-409).
__global__ void __launch_bounds__(kThreads) seed_kernel(const SeedParams p) {
    const int n = p.n;
    const uint64_t dim = 1ull << n;
    const uint32_t per_block = dim < kTileAmps ? uint32_t(dim) : uint32_t(kTileAmps);
    const uint32_t chunks = uint32_t(dim / per_block);
    const uint32_t s = blockIdx.x / chunks, chunk = blockIdx.x % chunks;
    const float2 *psi = p.psi + s * dim;
    float2 *lam = p.lam + s * dim;
    double e = 0.0;
    for (uint32_t k = threadIdx.x; k < per_block; k += kThreads) {
        const uint32_t x = chunk * per_block + k;
        const uint32_t t = x ^ uint32_t(p.x_mask);
        const float2 f = seed_factor(x, p.x_mask, p.z_mask, p.y_count, p.wfinal, p.czfinal);
        const float2 pt = psi[t], px = psi[x];
        const float2 l = cmul(f, pt);
        lam[x] = l;
        e += 0.5 * (double(px.x) * double(l.x) + double(px.y) * double(l.y));
    }
    // deterministic block reduction
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

// ---------------------------------------------------- sample-resident
// n <= 12: a tile holds 2^(12-n) whole samples, so the forward over every
// stage, the observable step and the adjoint backward run without leaving
// shared memory; HBM sees psi0, the checkpoint slots and nothing else.
__device__ __forceinline__ void tma_load3(void *dst, const CUtensorMap *map, uint64_t *bar,
                                          int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(su32(dst)),
                 "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2),
                 "r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void tma_store3(const CUtensorMap *map, const void *src, int c0,
                                           int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group"
                 " [%0, {%1, %2, %3}], [%4];" ::"l"(reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(su32(src))
                 : "memory");
}

__global__ void __launch_bounds__(kThreads, 2)
    resident_kernel(const __grid_constant__ ResidentParams p,
                    const __grid_constant__ CUtensorMap m_psi0,
                    const __grid_constant__ CUtensorMap m_slots,
                    const __grid_constant__ CUtensorMap m_out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    uint8_t *pt = smem, *lt = smem + kTileBytes;
    double *es = reinterpret_cast<double *>(smem + 2 * kTileBytes); // 4096 doubles
    uint8_t *tail = smem + 2 * kTileBytes + kTileAmps * sizeof(double);
    uint64_t *mbar = reinterpret_cast<uint64_t *>(tail);
    float2 *ry_s = reinterpret_cast<float2 *>(tail + 64); // [2][12]
    float2 *tcol_s = ry_s + 24;                            // [2][16]
    double *acc = reinterpret_cast<double *>(tcol_s + 32); // [8][12][8]
    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    const int n = p.n, S = p.stages;
    const uint32_t rot = (n >= 12) ? 0xFFFu : ((1u << n) - 1u);
    const uint32_t xmask = (n >= 12) ? 0xFFFu : ((1u << n) - 1u);
    const int spt = kTileAmps >> n; // samples per tile (>= 1)

    for (int i = tid; i < 8 * 12 * 8; i += kThreads) acc[i] = 0.0;
    if (tid == 0) {
        prefetch_map(&m_psi0);
        prefetch_map(&m_slots);
        mbar_init(&mbar[0], 1);
        fence_mbar_init();
    }
    __syncthreads();
    uint32_t phase = 0;
    auto load_stage = [&](int s) { // stage data into slot s & 1 (threads 0..27)
        const int sl = s & 1;
        if (tid < 12) ry_s[sl * 12 + tid] = (int(tid) < n) ? p.ry[size_t(s) * n + tid] : make_float2(1.f, 0.f);
        else if (tid < 28) tcol_s[sl * 16 + (tid - 12)] = p.tcol[size_t(s) * 16 + (tid - 12)];
    };
    auto stage_cz = [&](int s) -> const CzSet * {
        const int c = p.stage_cz[s];
        return c >= 0 ? p.czsets + c : nullptr;
    };

    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
        if (tid == 0) {
            mbar_expect_tx(&mbar[0], kTileBytes);
            tma_load3(pt, &m_psi0, &mbar[0], 0, t * 256, 0);
        }
        load_stage(0);
        mbar_wait(&mbar[0], phase);
        phase ^= 1u;
        __syncthreads();
        // ---------------- forward over all stages
        for (int s = 0; s < S; ++s) {
            const int sl = s & 1;
            const DiagCtx d = diag_ctx(tid, 0u, p.trow + size_t(s) * 256, nullptr, nullptr, stage_cz(s));
            phase_fwd<0>(pt, tid, rot, ry_s + sl * 12, true, d, tcol_s + sl * 16);
            __syncthreads();
            if (rot & 0xF0u) {
                phase_fwd<1>(pt, tid, rot, ry_s + sl * 12, false, d, tcol_s + sl * 16);
                __syncthreads();
            }
            if (rot & 0xF00u) phase_fwd<2>(pt, tid, rot, ry_s + sl * 12, false, d, tcol_s + sl * 16);
            if (s + 1 < S) load_stage(s + 1);
            const bool slot = ((s + 1) % p.ckpt == 0) && (s + 1 < S) && !p.forward_only;
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
        if (p.forward_only) {
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
#pragma unroll 4
        for (int j = 0; j < 16; ++j) {
            const uint32_t l = (tid << 4) | uint32_t(j);
            const uint32_t x = l & xmask;
            const uint32_t lp = l ^ uint32_t(p.x_mask);
            const float2 f = seed_factor(x, p.x_mask, p.z_mask, p.y_count, p.wfinal, p.czfinal);
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
        if (tid < uint32_t(spt)) {
            const uint64_t sample = uint64_t(t) * spt + tid;
            if (sample < p.batch) p.expect[sample] = es[tid << (n < 12 ? n : 12)];
        }
        // ---------------- backward
        if (S > 0) load_stage(S - 1);
        __syncthreads();
        for (int s = S - 1; s >= 0; --s) {
            const int sl = s & 1;
            if (((s + 1) % p.ckpt == 0) && (s + 1 < S)) { // re-anchor psi at the slot
                if (tid == 0) {
                    mbar_expect_tx(&mbar[0], kTileBytes);
                    tma_load3(pt, &m_slots, &mbar[0], 0, t * 256, (s + 1) / p.ckpt - 1);
                }
                mbar_wait(&mbar[0], phase);
                phase ^= 1u;
            }
            const DiagCtx d = diag_ctx(tid, 0u, p.trow + size_t(s) * 256, nullptr, nullptr, stage_cz(s));
            double *acc_w = acc + warp * 12 * 8;
            if (rot & 0xF00u) {
                phase_bwd<2>(pt, lt, tid, rot, rot, ry_s + sl * 12, false, d, tcol_s + sl * 16, acc_w);
                __syncthreads();
            }
            if (rot & 0xF0u) {
                phase_bwd<1>(pt, lt, tid, rot, rot, ry_s + sl * 12, false, d, tcol_s + sl * 16, acc_w);
                __syncthreads();
            }
            phase_bwd<0>(pt, lt, tid, rot, rot, ry_s + sl * 12, true, d, tcol_s + sl * 16, acc_w);
            if (s > 0) load_stage(s - 1);
            __syncthreads();
            if (tid < 96) {
                const int lb = tid >> 3, c = tid & 7;
                if (lb < n) {
                    double sum = 0.0;
#pragma unroll
                    for (int w = 0; w < 8; ++w) {
                        sum += acc[(w * 12 + lb) * 8 + c];
                        acc[(w * 12 + lb) * 8 + c] = 0.0;
                    }
                    double *dst = p.kpart + (size_t(blockIdx.x) * S + s) * size_t(n) * 8 + lb * 8 + c;
                    *dst += sum;
                }
            }
            __syncthreads();
        }
    }
    if (tid == 0) bulk_wait0();
}

// --------------------------------------------------- per-call θ prep
__device__ inline double2 zmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ inline double2 zconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ inline double2 zadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

struct M2 {
    double2 a, b, c, d; // [[a, b], [c, d]]
};
__device__ inline M2 mmul(const M2 &x, const M2 &y) {
    return {zadd(zmul(x.a, y.a), zmul(x.b, y.c)), zadd(zmul(x.a, y.b), zmul(x.b, y.d)),
            zadd(zmul(x.c, y.a), zmul(x.d, y.c)), zadd(zmul(x.c, y.b), zmul(x.d, y.d))};
}
__device__ inline M2 mdag(const M2 &x) { return {zconj(x.a), zconj(x.c), zconj(x.b), zconj(x.d)}; }
// rotation_matrix / rotation_derivative, circuit.cpp:61-87.
__device__ inline M2 rot_m(int axis, double theta, bool deriv) {
    double s, c;
    sincos(theta / 2.0, &s, &c);
    double a = c, b = s;
    if (deriv) {
        a = -0.5 * s;
        b = 0.5 * c;
    }
    switch (axis) {
    case 0: return {{a, 0}, {0, -b}, {0, -b}, {a, 0}};
    case 1: return {{a, 0}, {-b, 0}, {b, 0}, {a, 0}};
    default: return {{a, -b}, {0, 0}, {0, 0}, {a, b}};
    }
}
__device__ inline M2 hadamard() {
    const double r = 0.70710678118654752440;
    return {{r, 0}, {r, 0}, {r, 0}, {-r, 0}};
}
__device__ inline M2 sec_gate(uint32_t enc, const double *theta, bool deriv) {
    const uint32_t kind = enc & 3u;
    if (kind == kSecH) return hadamard();
    return rot_m(int(kind), theta[enc >> 2], deriv);
}

// One thread per section: compose the run's 2x2 in fp64, decompose
// U = e^{i delta} Rz(alpha) Ry(beta) Rz(gamma) and scatter the stage data.
__global__ void prep_sections_kernel(int n_sec, const uint32_t *sec_q, const uint32_t *sec_stage,
                                     const uint32_t *sec_alpha_row, const uint32_t *sec_off,
                                     const uint32_t *sec_gates, const double *theta, int n,
                                     float2 *ry, double *wg, double *wa, double *sec_gamma) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_sec) return;
    M2 u{{1, 0}, {0, 0}, {0, 0}, {1, 0}};
    for (uint32_t k = sec_off[i]; k < sec_off[i + 1]; ++k) u = mmul(sec_gate(sec_gates[k], theta, false), u);
    // normalise to SU(2): v = u / sqrt(det u)
    const double2 det = zadd(zmul(u.a, u.d), make_double2(-(u.b.x * u.c.x - u.b.y * u.c.y),
                                                          -(u.b.x * u.c.y + u.b.y * u.c.x)));
    const double dr = sqrt(hypot(det.x, det.y)), dth = 0.5 * atan2(det.y, det.x);
    const double2 inv = make_double2(cos(dth) / dr, -sin(dth) / dr);
    const double2 a = zmul(u.a, inv), b = zmul(u.c, inv);
    const double ca = hypot(a.x, a.y), cb = hypot(b.x, b.y);
    const double beta = 2.0 * atan2(cb, ca);
    double alpha, gamma;
    if (cb < 1e-13) {
        alpha = 0.0;
        gamma = -2.0 * atan2(a.y, a.x);
    } else if (ca < 1e-13) {
        alpha = 2.0 * atan2(b.y, b.x);
        gamma = 0.0;
    } else {
        const double ga = atan2(a.y, a.x), gb = atan2(b.y, b.x);
        alpha = gb - ga;
        gamma = -ga - gb;
    }
    const uint32_t q = sec_q[i], st = sec_stage[i];
    double sb, cbt;
    sincos(0.5 * beta, &sb, &cbt);
    ry[size_t(st) * n + q] = make_float2(float(cbt), float(sb));
    wg[size_t(st) * n + q] = gamma;
    wa[size_t(sec_alpha_row[i]) * n + q] = alpha;
    sec_gamma[i] = gamma;
}

// Per stage: e^{i sum w_b x_b} tables for pass-A columns (q0..3), rows
// (q4..11) and tile bits (q12..19, q20..27), fp64 -> complex64.
__global__ void diag_tables_kernel(int stages, int n, const double *wg, const double *wa,
                                   float2 *tcol, float2 *trow, float2 *tt1, float2 *tt2,
                                   double *wfinal) {
    const int s = blockIdx.x;
    if (s == stages) {
        for (int q = threadIdx.x; q < n; q += blockDim.x)
            wfinal[q] = wg[size_t(stages) * n + q] + wa[size_t(stages) * n + q];
        return;
    }
    for (int e = threadIdx.x; e < 16 + 3 * 256; e += blockDim.x) {
        int base, bits, idx;
        float2 *dst;
        if (e < 16) { base = 0; bits = 4; idx = e; dst = tcol + size_t(s) * 16 + idx; }
        else if (e < 272) { base = 4; bits = 8; idx = e - 16; dst = trow + size_t(s) * 256 + idx; }
        else if (e < 528) { base = 12; bits = 8; idx = e - 272; dst = tt1 + size_t(s) * 256 + idx; }
        else { base = 20; bits = 8; idx = e - 528; dst = tt2 + size_t(s) * 256 + idx; }
        double ang = 0.0;
        for (int b = 0; b < bits; ++b) {
            const int q = base + b;
            if (q < n && ((idx >> b) & 1)) ang += wg[size_t(s) * n + q] + wa[size_t(s) * n + q];
        }
        double sn, cs;
        sincos(ang, &sn, &cs);
        *dst = make_float2(float(cs), float(sn));
    }
}

// kout[e] = sum over CTAs (fixed order) of kpart[cta][e]; expect[s] = sum of
// the seed kernel's chunk partials.
__global__ void reduce_kernel(long long entries, int grid, const double *kpart, double *kout,
                              const double *epart, int chunks, uint32_t batch, double *expect) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < entries) {
        double s = 0.0;
        for (int g = 0; g < grid; ++g) s += kpart[size_t(g) * entries + i];
        kout[i] = s;
    }
    if (epart && i < batch) {
        double s = 0.0;
        for (int c = 0; c < chunks; ++c) s += epart[size_t(i) * chunks + c];
        expect[i] = s;
    }
}

// One thread per section: K at the point before Ry(beta) -> K at the run
// start (Rz(gamma)^dag), then walk the run's gates: grad = Re Tr(dg K g^dag),
// K <- g K g^dag. Last block: loss = sum_s E_s (engine.cpp:733-738).
__global__ void finalize_kernel(int n_sec, const uint32_t *sec_q, const uint32_t *sec_stage,
                                const uint32_t *sec_off, const uint32_t *sec_gates,
                                const double *sec_gamma, const double *theta, int n,
                                const double *kout, double *grad, const double *expect,
                                uint32_t batch, double *loss) {
    if (blockIdx.x == gridDim.x - 1) {
        if (threadIdx.x < 32) {
            double s = 0.0;
            for (uint32_t i = threadIdx.x; i < batch; i += 32) s += expect[i];
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
            if (threadIdx.x == 0) *loss = s;
        }
        return;
    }
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_sec) return;
    const double *k = kout + (size_t(sec_stage[i]) * n + sec_q[i]) * 8;
    const double g = sec_gamma[i];
    const double2 e = make_double2(cos(g), sin(g));
    M2 K{{k[0], k[1]}, zmul(make_double2(k[2], k[3]), e), zmul(make_double2(k[4], k[5]), zconj(e)),
         {k[6], k[7]}};
    for (uint32_t j = sec_off[i]; j < sec_off[i + 1]; ++j) {
        const uint32_t enc = sec_gates[j];
        const M2 gm = sec_gate(enc, theta, false);
        if ((enc & 3u) != kSecH) {
            const M2 dg = sec_gate(enc, theta, true);
            const M2 t = mmul(mmul(dg, K), mdag(gm));
            grad[enc >> 2] = t.a.x + t.d.x;
        }
        K = mmul(mmul(gm, K), mdag(gm));
    }
}

// ------------------------------------------ per-gate (unfused) comparator
// One HBM traversal per gate: apply_rotation_kernel / apply_cz_kernel /
// apply_cnot_kernel (engine.cpp:111-202) and rotation_backward_kernel
// (engine.cpp:207-256), psi uncomputed in place instead of a stored ledger.
__device__ __forceinline__ void pair_apply_f(int axis, float c, float s, float2 &a, float2 &b) {
    const float2 A = a, Bv = b;
    switch (axis) {
    case 0:
        a = make_float2(c * A.x + s * Bv.y, c * A.y - s * Bv.x);
        b = make_float2(c * Bv.x + s * A.y, c * Bv.y - s * A.x);
        break;
    case 1:
        a = make_float2(c * A.x - s * Bv.x, c * A.y - s * Bv.y);
        b = make_float2(s * A.x + c * Bv.x, s * A.y + c * Bv.y);
        break;
    default:
        a = make_float2(c * A.x + s * A.y, c * A.y - s * A.x);
        b = make_float2(c * Bv.x - s * Bv.y, c * Bv.y + s * Bv.x);
        break;
    }
}

__global__ void __launch_bounds__(256) gate_fwd_kernel(float2 *psi, int n, uint64_t total_pairs,
                                                       int kind, int axis, uint32_t q0, uint32_t q1,
                                                       const double *theta, uint32_t param) {
    float c = 1.f, s = 0.f;
    if (kind == 0) {
        double sd, cd;
        sincos(theta[param] / 2.0, &sd, &cd);
        c = float(cd);
        s = float(sd);
    }
    const uint64_t half = 1ull << (n - 1);
    const uint32_t tq = kind == 0 ? q0 : q1;
    const uint64_t mask = 1ull << tq, lo = mask - 1;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total_pairs;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t smp = i / half, k = i % half;
        float2 *base = psi + (smp << n);
        const uint64_t i0 = ((k & ~lo) << 1) | (k & lo), i1 = i0 | mask;
        float2 a = base[i0], b = base[i1];
        if (kind == 0) {
            pair_apply_f(axis, c, s, a, b);
        } else if (kind == 1) { // CZ(q0,q1): -1 on |..1..1..> (target bit q1 = 1 in i1)
            if ((i1 >> q0) & 1ull) b = make_float2(-b.x, -b.y);
        } else { // CNOT: swap the pair when the control is set
            if ((i0 >> q0) & 1ull) {
                const float2 t = a;
                a = b;
                b = t;
            }
        }
        base[i0] = a;
        base[i1] = b;
    }
}

__global__ void __launch_bounds__(256) gate_bwd_kernel(float2 *psi, float2 *lam, int n,
                                                       uint64_t total_pairs, int kind, int axis,
                                                       uint32_t q0, uint32_t q1,
                                                       const double *theta, uint32_t param,
                                                       double *gpart) {
    float c = 1.f, s = 0.f;
    double sd = 0, cd = 1;
    if (kind == 0) {
        sincos(theta[param] / 2.0, &sd, &cd);
        c = float(cd);
        s = float(sd);
    }
    const float dc = float(-0.5 * sd), ds = float(0.5 * cd);
    const uint64_t half = 1ull << (n - 1);
    const uint32_t tq = kind == 0 ? q0 : q1;
    const uint64_t mask = 1ull << tq, lo = mask - 1;
    double acc = 0.0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total_pairs;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t smp = i / half, k = i % half;
        float2 *pb = psi + (smp << n), *lb = lam + (smp << n);
        const uint64_t i0 = ((k & ~lo) << 1) | (k & lo), i1 = i0 | mask;
        float2 a = pb[i0], b = pb[i1], la = lb[i0], lbv = lb[i1];
        if (kind == 0) {
            pair_apply_f(axis, c, -s, a, b); // psi_in = u^dag psi_out
            float2 wa = a, wb = b;
            pair_apply_f(axis, dc, ds, wa, wb); // du psi_in
            acc += double(la.x) * wa.x + double(la.y) * wa.y + double(lbv.x) * wb.x +
                   double(lbv.y) * wb.y;
            pair_apply_f(axis, c, -s, la, lbv);
        } else if (kind == 1) {
            if ((i1 >> q0) & 1ull) {
                b = make_float2(-b.x, -b.y);
                lbv = make_float2(-lbv.x, -lbv.y);
            }
        } else {
            if ((i0 >> q0) & 1ull) {
                float2 t = a; a = b; b = t;
                t = la; la = lbv; lbv = t;
            }
        }
        pb[i0] = a;
        pb[i1] = b;
        lb[i0] = la;
        lb[i1] = lbv;
    }
    if (kind == 0) {
        __shared__ double red[8];
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < 8; ++w) t += red[w];
            gpart[blockIdx.x] = t;
        }
    }
}

__global__ void gate_grad_reduce_kernel(const double *gpart, int gblocks, const uint32_t *params,
                                        int n_rot, double *grad) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rot) return;
    double s = 0.0;
    for (int b = 0; b < gblocks; ++b) s += gpart[size_t(r) * gblocks + b];
    grad[params[r]] = s;
}

} // namespace

// ================================================================ launchers
size_t pass_smem_bytes(bool backward) { return PassSmem::bytes(backward); }
size_t resident_smem_bytes() {
    return size_t(2) * kTileBytes + size_t(kTileAmps) * sizeof(double) + 64 + 2 * 12 * 8 +
           2 * 16 * 8 + 8 * 12 * 8 * 8 + 1024;
}

static bool g_attr_done = false;
static cudaError_t ensure_attrs() {
    if (g_attr_done) return cudaSuccess;
    cudaError_t e;
    e = cudaFuncSetAttribute(pass_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(pass_smem_bytes(false)));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(pass_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(pass_smem_bytes(true)));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(resident_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(resident_smem_bytes()));
    if (e != cudaSuccess) return e;
    g_attr_done = true;
    return cudaSuccess;
}

int pass_occupancy(bool backward) {
    if (ensure_attrs() != cudaSuccess) return 0;
    int blocks = 0;
    if (backward)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, pass_kernel<true>, kThreads,
                                                      pass_smem_bytes(true));
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, pass_kernel<false>, kThreads,
                                                      pass_smem_bytes(false));
    return blocks;
}
int resident_occupancy() {
    if (ensure_attrs() != cudaSuccess) return 0;
    int blocks = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, resident_kernel, kThreads,
                                                  resident_smem_bytes());
    return blocks;
}

cudaError_t launch_pass(cudaStream_t st, bool backward, int grid, const PassParams &p,
                        const CUtensorMap *psi_in, const CUtensorMap *psi_out,
                        const CUtensorMap *lam) {
    cudaError_t e = ensure_attrs();
    if (e != cudaSuccess) return e;
    const CUtensorMap &l = lam ? *lam : *psi_out;
    if (backward)
        pass_kernel<true><<<grid, kThreads, pass_smem_bytes(true), st>>>(p, *psi_in, *psi_out, l);
    else
        pass_kernel<false><<<grid, kThreads, pass_smem_bytes(false), st>>>(p, *psi_in, *psi_out, l);
    return cudaGetLastError();
}

cudaError_t launch_resident(cudaStream_t st, int grid, const ResidentParams &p,
                            const CUtensorMap *psi0, const CUtensorMap *slots_map,
                            const CUtensorMap *out_map) {
    cudaError_t e = ensure_attrs();
    if (e != cudaSuccess) return e;
    resident_kernel<<<grid, kThreads, resident_smem_bytes(), st>>>(p, *psi0, *slots_map, *out_map);
    return cudaGetLastError();
}

cudaError_t launch_seed(cudaStream_t st, const SeedParams &p) {
    const uint64_t dim = 1ull << p.n;
    const uint64_t per_block = dim < kTileAmps ? dim : kTileAmps;
    const uint64_t blocks = (dim / per_block) * p.batch;
    seed_kernel<<<unsigned(blocks), kThreads, 0, st>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_prep_sections(cudaStream_t st, int n_sec, const uint32_t *sec_q,
                                 const uint32_t *sec_stage, const uint32_t *sec_alpha_row,
                                 const uint32_t *sec_off, const uint32_t *sec_gates,
                                 const double *theta, int n, float2 *ry, double *wg, double *wa,
                                 double *sec_gamma) {
    if (n_sec == 0) return cudaSuccess;
    prep_sections_kernel<<<(n_sec + 127) / 128, 128, 0, st>>>(
        n_sec, sec_q, sec_stage, sec_alpha_row, sec_off, sec_gates, theta, n, ry, wg, wa, sec_gamma);
    return cudaGetLastError();
}

cudaError_t launch_diag_tables(cudaStream_t st, int stages, int n, const double *wg,
                               const double *wa, float2 *tcol, float2 *trow, float2 *tt1,
                               float2 *tt2, double *wfinal) {
    diag_tables_kernel<<<stages + 1, 256, 0, st>>>(stages, n, wg, wa, tcol, trow, tt1, tt2, wfinal);
    return cudaGetLastError();
}

cudaError_t launch_reduce(cudaStream_t st, long long entries, int grid, const double *kpart,
                          double *kout, const double *epart, int chunks, uint32_t batch,
                          double *expect) {
    const long long work = entries > (long long)batch ? entries : (long long)batch;
    if (work == 0) return cudaSuccess;
    reduce_kernel<<<unsigned((work + 255) / 256), 256, 0, st>>>(entries, grid, kpart, kout, epart,
                                                                chunks, batch, expect);
    return cudaGetLastError();
}

cudaError_t launch_finalize(cudaStream_t st, int n_sec, const uint32_t *sec_q,
                            const uint32_t *sec_stage, const uint32_t *sec_off,
                            const uint32_t *sec_gates, const double *sec_gamma,
                            const double *theta, int n, const double *kout, double *grad,
                            const double *expect, uint32_t batch, double *loss) {
    const int blocks = (n_sec + 127) / 128 + 1;
    finalize_kernel<<<blocks, 128, 0, st>>>(n_sec, sec_q, sec_stage, sec_off, sec_gates, sec_gamma,
                                            theta, n, kout, grad, expect, batch, loss);
    return cudaGetLastError();
}

int gate_grid(uint64_t pairs) {
    uint64_t b = (pairs + 255) / 256;
    if (b > 148 * 8) b = 148 * 8;
    return int(b ? b : 1);
}

cudaError_t launch_gate_fwd(cudaStream_t st, float2 *psi, int n, uint32_t batch, int kind,
                            int axis, uint32_t q0, uint32_t q1, const double *theta,
                            uint32_t param) {
    const uint64_t pairs = (uint64_t(batch) << n) / 2;
    gate_fwd_kernel<<<gate_grid(pairs), 256, 0, st>>>(psi, n, pairs, kind, axis, q0, q1, theta, param);
    return cudaGetLastError();
}

cudaError_t launch_gate_bwd(cudaStream_t st, float2 *psi, float2 *lam, int n, uint32_t batch,
                            int kind, int axis, uint32_t q0, uint32_t q1, const double *theta,
                            uint32_t param, double *gpart) {
    const uint64_t pairs = (uint64_t(batch) << n) / 2;
    gate_bwd_kernel<<<gate_grid(pairs), 256, 0, st>>>(psi, lam, n, pairs, kind, axis, q0, q1, theta,
                                                      param, gpart);
    return cudaGetLastError();
}

cudaError_t launch_gate_grad_reduce(cudaStream_t st, const double *gpart, int gblocks,
                                    const uint32_t *params, int n_rot, double *grad) {
    if (n_rot == 0) return cudaSuccess;
    gate_grad_reduce_kernel<<<(n_rot + 127) / 128, 128, 0, st>>>(gpart, gblocks, params, n_rot, grad);
    return cudaGetLastError();
}

} // namespace qfb
