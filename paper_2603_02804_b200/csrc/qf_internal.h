// Internal structures shared by the host planner (qf_plan.cpp, qf_capi.cpp)
// and the sm_100a kernels (qf_pass.cu, qf_resident.cu, qf_prep.cu,
// qf_pergate.cu). Not part of the C-ABI.
#pragma once

#include <atomic>
#include <cstddef>
#include <cstdint>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/qfuse_b200.h"

namespace qfb {

// ---------------------------------------------------------------- geometry
// One tile = 4096 amplitudes (32 KiB of complex64) held in shared memory as
// 256 rows x 16 amplitudes (128 B) with the TMA 128B swizzle. Local index l
// (12 bits): bits 0..3 = column = global qubits 0..3; bits 4..11 = rows = a
// contiguous block of 8 qubits starting at the layout's row_start (n > 12),
// or qubits 4..11 and then sample bits (n <= 12, the sample-resident layout).
// A thread of a *group phase* G holds local bits [4G, 4G+4) in 16 registers;
// the other 8 local bits form its thread index tau (in bit order).
constexpr int kTileBits = 12;
constexpr int kTileAmps = 1 << kTileBits;
constexpr int kTileBytes = kTileAmps * 8;
constexpr int kThreads = 256;
constexpr int kMaxQubits = 28;

// Encoded section gate: bits 0..1 kind (0 Rx, 1 Ry, 2 Rz, 3 fixed H), bits 2.. param.
constexpr uint32_t kSecH = 3u;

// Diagonal D_s(x) = (-1)^{Q(x)} e^{i sum_q w_q x_q} of one stage, tabulated in
// the layout of the pass that applies it: register bits of the diag group
// (treg), the thread bits (tthr), tile bits 0..7 / 8..15 (tt1, tt2).
struct DiagTab {
    float2 treg[16];
    float2 tthr[256];
    float2 tt1[256];
    float2 tt2[256];
};

// A CZ set (quadratic form Q) in one layout/diag group (theta-independent).
// sign bit of register j for thread tau in tile tb:
//   sbase = Q(tile) ^ Q(thr) ^ parity(tau & Rtile), M = Mtile ^ Mthr,
//   sgn   = (sbase ? 0xFFFF : 0) ^ qreg ^ linmask(M)
// thrinfo[tau] = Q(thr) << 4 | Mthr;  tileinfo[tb] = Q(tile) | Mtile << 1 | Rtile << 8.
struct CzTab {
    uint32_t qreg;
    uint32_t pad[3];
    uint16_t thrinfo[256];
};

// Wide-group view of layout A (forward passes, qf_pass_wide.cu): a thread holds
// 64 amplitudes, the 6 local bits {0,1,2,3,7,8} (group L) or {4,5,6,9,10,11}
// (group H) in registers. The diagonal is applied in group L: its register bits
// (treg[64]) and the 6 thread bits (tthr[64]); the tile terms are DiagTab's.
__host__ __device__ constexpr int wide_reg_bit(int b) { return b < 4 ? b : b + 3; } // 0,1,2,3,7,8
__host__ __device__ constexpr int wide_thr_bit(int b) { return b < 3 ? b + 4 : b + 6; } // 4,5,6,9,10,11
struct DiagTabW {
    float2 treg[64];
    float2 tthr[64];
};
// CZ signs in the wide L view: sgn (64 bits) = (sbase ? ~0 : 0) ^ qreg ^ linmask6(M),
// sbase = Q(tile) ^ Q(thr) ^ parity(tau & Rtile), M = Mtile ^ Mthr;
// thrinfo[tau] = Q(thr) << 6 | Mthr;  tileinfo[tb] = Q(tile) | Mtile << 1 | Rtile << 8.
struct CzTabW {
    unsigned long long qreg;
    uint16_t thrinfo[64];
};

// Adjacency of a CZ set, for the observable fold (seed).
struct CzAdj {
    uint32_t adjlo[32]; // bit p < q of adjlo[q] = CZ(p, q)
};

// One fused HBM pass over the batch store. It applies, in shared memory, up
// to two Ry rounds on its resident qubits with the stage diagonal between
// them:  Ry_{s0}(X) -> D -> Ry_{s1}(X)  (forward), or the inverse with K
// accumulation (backward). ops per phase: bit 0 = round 0, 1 = diag, 2 = round 1.
struct PassPhase {
    int8_t g;
    uint8_t ops;
};
// Compile-time program of a pass (qf_device.cuh prog_*): 0 = none.
constexpr uint32_t prog_encode(int nph, const PassPhase *ph, uint32_t rot_mask) {
    uint32_t v = uint32_t(nph) & 7u;
    for (int g = 0; g < 3; ++g)
        if (((rot_mask >> (4 * g)) & 0xFu) == 0xFu) v |= 1u << (3 + g);
    for (int i = 0; i < nph; ++i) v |= (uint32_t(ph[i].g) | (uint32_t(ph[i].ops) << 2)) << (6 + 5 * i);
    return v;
}
// The programs compiled as straight-line kernels: interior passes of layout A
// (12 rotated qubits, diagonal in group 0) and of layout B at n = 20 (groups
// 1, 2) and n = 16 (group 2 only).
constexpr PassPhase kProgAPh[5] = {{2, 1}, {1, 1}, {0, 7}, {1, 4}, {2, 4}};
constexpr PassPhase kProgB20Ph[3] = {{1, 1}, {2, 7}, {1, 4}};
constexpr PassPhase kProgB16Ph[1] = {{2, 7}};
// n = 16 with the column group moved to layout B (qf_plan.cpp): A runs kProgB20's
// phases on groups 1, 2; B rotates groups 0 and 2.
constexpr PassPhase kProgB16xPh[3] = {{0, 1}, {2, 7}, {0, 4}};
constexpr uint32_t kProgA = prog_encode(5, kProgAPh, 0xFFFu);
constexpr uint32_t kProgB20 = prog_encode(3, kProgB20Ph, 0xFF0u);
constexpr uint32_t kProgB16 = prog_encode(1, kProgB16Ph, 0xF00u);
constexpr uint32_t kProgB16x = prog_encode(3, kProgB16xPh, 0xF0Fu);
// Balanced two-layout schedule (n = 20): the column group's Ry of stage s is
// applied by the pass that applies D_s, so both layouts run round 0 on their 8
// row qubits and round 1 on rows + columns (4 phases, 20 Ry each).
constexpr PassPhase kProgAltPh[4] = {{1, 1}, {2, 7}, {1, 4}, {0, 4}};
constexpr uint32_t kProgAlt = prog_encode(4, kProgAltPh, 0xFFFu);
// 17 <= n <= 19: layout B rotates only some of group 1's row bits (runtime bit
// checks in that group; the encoding keeps the FULL flags, not the bit pattern)
constexpr uint32_t kProgB20P = prog_encode(3, kProgB20Ph, 0xF20u);
constexpr uint32_t kProgAltP = prog_encode(4, kProgAltPh, 0xF2Fu);
// 13 <= n <= 15: layout B rotates the columns and only part of group 2 (qubits 12..n-1)
constexpr uint32_t kProgB16xP = prog_encode(3, kProgB16xPh, 0x20Fu);

struct PassParams {
    int n;
    int tiles;
    int tile_lo_bits;  // tile bits between the column and the rows (row_start - 4)
    int tile_hi_bits;  // tile bits above the rows (n - row_start - 8)
    uint32_t rot_mask; // local bits rotated by this pass (rot0 | rot1)
    uint32_t rot0, rot1; // ... in round 0 / round 1 (they differ in the balanced backward)
    int qmap[12];      // local bit -> qubit
    int s0, s1;        // stages of rounds 0 / 1 (-1 = absent)
    int nph;
    PassPhase ph[6];
    int gd;            // group phase that applies the diagonal
    const float2 *ry;  // [stages][n] (cos, sin) of beta/2
    const DiagTab *dt; // diagonal of this pass (nullptr = none)
    const CzTab *cz;   // its CZ set in this layout (nullptr = none)
    const uint32_t *tileinfo;
    // wide-group forward of layout A (nullptr: not available for this pass)
    const DiagTabW *dtw;
    const CzTabW *czw;
    const uint32_t *tileinfow;
    int write_psi;     // backward: store psi (0 when the next reader is a slot)
    int zmask;         // backward: bit r = round r measures Z (its stage is 0)
    uint32_t prog;     // prog_encode(nph, ph, rot_mask)
    int l2pf;          // backward light passes: L2 prefetch of the next ring load
    double *kpart;     // backward: [grid][stages][n][8]
    long long kstride; // stages*n*8
    uint32_t *slot16;  // MemSave: the pass also writes its output as bf16 pairs here (wide forward)
};

// n <= 12: a tile holds 2^(12-n) whole samples; every stage runs in smem.
struct ResidentParams {
    int n;
    int stages;
    int ckpt; // re-anchor the uncompute every ckpt stages
    int tiles;
    uint32_t batch;
    uint64_t x_mask, z_mask;
    uint32_t y_count;
    const float2 *ry;          // [stages][n]
    const DiagTab *dt;         // [stages]
    const CzTab *cztabs;       // [CZ set][cz_stride] tables (per resident layout)
    int cz_stride;             // resident layouts: 1, or 2 for n = 12 (diagonal in group 0 / 2)
    const int *stage_cz;       // [stages] -> CZ set index or -1
    const double *wfinal;      // [n] final diagonal phases
    const CzAdj *czfinal;      // nullptr = none
    double *kpart;             // [grid][stages][n][8]
    double *expect;            // [batch]
    int forward_only;          // forward, fold D_f, store the final state
};

struct SeedParams {
    int n;
    uint32_t batch;
    uint64_t x_mask, z_mask;
    uint32_t y_count;
    const double *wfinal;
    const CzAdj *czfinal;
    const float2 *psi;
    float2 *lam;
    double *epart;  // [batch][chunks]
    int apply_only; // 1: lam = D_f psi (forward-state readout), no observable
};

// ------------------------------------------------------------- launchers
cudaError_t launch_prep_sections(cudaStream_t st, int n_sec, const uint32_t *sec_q,
                                 const uint32_t *sec_stage, const uint32_t *sec_alpha_row,
                                 const uint32_t *sec_off, const uint32_t *sec_gates,
                                 const double *theta, int n, float2 *ry, double *wg,
                                 double *wa, double *sec_gamma, double *sec_phase);
// Forward-state readout: wfinal[n] = the global phase e^{i sum delta} the stage
// model drops (it cancels in <O> and every gradient, not in the state itself).
cudaError_t launch_phase_sum(cudaStream_t st, int n_sec, const double *sec_phase, int n,
                             double *wfinal);
// dq: [layouts][28] qubit of (reg 0..3, thr 0..7, tile 0..15), -1 = none.
cudaError_t launch_diag_tables(cudaStream_t st, int stages, int n, const double *wg,
                               const double *wa, const int *stage_layout, const int *dq,
                               DiagTab *dt, double *wfinal);
// Wide-group tables of the stages layout 0 applies (stage_layout[s] == 0), from the
// wide view dqw[0..5] reg bits, [6..11] thread bits (qubits, -1 = none).
cudaError_t launch_diag_tables_wide(cudaStream_t st, int stages, int n, const double *wg,
                                    const double *wa, const int *stage_layout, const int *dqw,
                                    DiagTabW *dtw);
int wide_grid(int sms);
// The forward pass runs the wide kernel (interior layout-A pass with wide tables);
// its grid is wide_grid(sms) instead of the narrow kernels' occupancy x sms.
bool pass_is_wide(bool backward, const PassParams &p);
// A pass with this phase-program code runs a compiled straight-line instance
// (launch_pass); otherwise the runtime-dispatch kernel.
bool prog_compiled(bool backward, uint32_t prog);
cudaError_t launch_pass_wide(cudaStream_t st, int grid, const PassParams &p, const CUtensorMap *psi_in,
                             const CUtensorMap *psi_out);
cudaError_t launch_pass(cudaStream_t st, bool backward, int grid, const PassParams &p,
                        const CUtensorMap *psi_in, const CUtensorMap *psi_out,
                        const CUtensorMap *lam);
cudaError_t launch_resident(cudaStream_t st, int grid, const ResidentParams &p,
                            const CUtensorMap *psi0, const CUtensorMap *slots_map,
                            const CUtensorMap *out_map);
cudaError_t launch_seed(cudaStream_t st, const SeedParams &p);
cudaError_t launch_reduce(cudaStream_t st, long long entries, int grid, const double *kpart,
                          double *kout, const double *epart, int chunks, uint32_t batch,
                          double *expect);
cudaError_t launch_finalize(cudaStream_t st, int n_sec, const uint32_t *sec_q,
                            const uint32_t *sec_stage, const uint32_t *sec_off,
                            const uint32_t *sec_gates, const double *sec_gamma,
                            const double *theta, int n, const double *kout, double *grad,
                            const double *expect, uint32_t batch, double *loss);
cudaError_t launch_random_state(cudaStream_t st, uint64_t seed, uint64_t first_sample, int n,
                                uint32_t batch, double *scratch, float2 *out);
// Z of every (stage >= 1, qubit) from the previous stage's (X, Z) and Ry angle
// (qf_device.cuh kmeasure): streaming plans measure Z at stage 0 only.
cudaError_t launch_zchain(cudaStream_t st, int stages, int n, const float2 *ry, double *kout);
// StorageMode::MemSave slots: complex64 <-> bfloat16 pairs (uint32 per amplitude).
cudaError_t launch_narrow_bf16(cudaStream_t st, const float2 *src, uint32_t *dst, uint64_t amps);
cudaError_t launch_widen_bf16(cudaStream_t st, const uint32_t *src, float2 *dst, uint64_t amps);
int pass_occupancy(bool backward);
int resident_occupancy();
size_t pass_smem_bytes(bool backward);
size_t resident_smem_bytes();

// Per-gate (unfused) comparator kernels.
cudaError_t launch_gate_fwd(cudaStream_t st, float2 *psi, int n, uint32_t batch, int kind,
                            int axis, uint32_t q0, uint32_t q1, const double *theta,
                            uint32_t param);
cudaError_t launch_gate_bwd(cudaStream_t st, float2 *psi, float2 *lam, int n, uint32_t batch,
                            int kind, int axis, uint32_t q0, uint32_t q1, const double *theta,
                            uint32_t param, double *gpart);
cudaError_t launch_gate_grad_reduce(cudaStream_t st, const double *gpart, int gblocks,
                                    const uint32_t *params, int n_rot, double *grad);
int gate_grid(uint64_t pairs);

// complex128 path (qf_c128.cu): per-gate fp64 kernels.
int c128_gate_grid(uint64_t pairs);
cudaError_t launch_gate_fwd_c128(cudaStream_t st, double2 *psi, int n, uint32_t batch, int kind,
                                 int axis, uint32_t q0, uint32_t q1, const double *theta,
                                 uint32_t param);
cudaError_t launch_gate_bwd_c128(cudaStream_t st, double2 *psi, double2 *lam, int n, uint32_t batch,
                                 int kind, int axis, uint32_t q0, uint32_t q1, const double *theta,
                                 uint32_t param, double *gpart);
cudaError_t launch_seed_c128(cudaStream_t st, int n, uint32_t batch, uint64_t x_mask, uint64_t z_mask,
                             uint32_t y_count, const double2 *psi, double2 *lam, uint32_t chunks,
                             double *epart);
cudaError_t launch_reduce_c128(cudaStream_t st, const double *gpart, int gblocks,
                               const uint32_t *params, int n_rot, double *grad, const double *epart,
                               uint32_t chunks, uint32_t batch, double *expect, double *loss);

// complex128 fused path (qf_c128_fused.cu). The circuit becomes a list of ops —
// a *section* (maximal run of consecutive rotations on one qubit, one 2x2
// unitary), a CZ run (one diagonal), a CNOT — cut into *segments*: op ranges
// whose non-diagonal targets fit one shared-memory tile of 2^m amplitudes
// (m = min(n, 11), local qubits 0..2 always included for coalescing). A segment
// is one HBM pass. Inside it the ops are grouped into *rounds*: up to three
// sections (on at most three local bits) and any CZ runs between them are applied
// to eight register-resident amplitudes per thread between two shared-memory
// transposes; a CNOT is a round of its own. The backward measures, per section,
// X = Im(K01 + K10), Y = Re(K01 - K10), Z = Im(K00 - K11) of K = sum psi_in lam_in^dag
// and the gradient of rotation j is (1/2)(hx X + hy Y + hz Z), H_j = sum_m h_m sigma_m
// = B_j^dag g_j^dag P_j g_j B_j (c128_finalize).
constexpr int kC128TileBits = 11;
constexpr int kC128MaxSec = 32;      // sections per segment (shared K accumulators)
constexpr int kC128MaxOps = 64;      // ops per segment (staged in shared memory)
constexpr int kC128MaxRounds = 64;   // rounds per segment
constexpr int kC128MaxCzPairs = 128; // CZ pairs per segment (staged in shared memory)
constexpr int kC128RoundSecs = 3;    // sections per octet round (K accumulator slots)
constexpr int kC128SecWords = 8;     // double2 per section in secU (c128_prep)
struct C128Op {
    uint32_t type; // 0 section, 1 CZ run, 2 CNOT
    uint32_t q;    // section: register bit in its round | CZ run: Q of the round's octet offsets
                   // (bit j = parity of the run's pairs inside offset j) | CNOT: target qubit
    uint32_t a;    // section: index (plan-wide) | CZ run: first pair (plan-wide) | CNOT: control qubit
    uint32_t b;    // section: K slot in its round | CZ run: pair count
};
struct C128Round {
    uint32_t kind;     // 0 octet round (sections / CZ runs), 1 CNOT
    uint32_t op_begin, op_end;
    uint32_t nsec;     // sections in the round (<= kC128RoundSecs)
    uint32_t has_cz;   // the round applies a CZ run (needs the amplitudes' global indices)
    uint8_t bits[4];   // octet: local positions of the register bits (ascending)
    uint8_t gq[4];     // ... and their qubits
    uint8_t sec[4];    // section (index within the segment) of K slot s
    uint8_t sbit[4];   // register bit of K slot s
};
struct C128Seg {
    uint32_t m, nrest, op_begin, op_end, sec_begin, nsec, cz_begin, cz_count, round_begin, round_end;
    int8_t lpos[32]; // qubit -> local bit, -1 if the qubit indexes tiles
    uint8_t lq[16];  // local bit -> qubit (ascending)
    uint8_t rq[32];  // tile bit -> qubit (ascending)
};
struct C128Plan {
    std::vector<C128Op> ops;
    std::vector<C128Round> rounds;
    std::vector<C128Seg> segs;
    std::vector<uint32_t> cz;        // q0 | q1 << 8
    std::vector<uint32_t> sec_off, sec_cnt, sec_gates; // gates: axis | param << 2
};
C128Plan build_c128_plan(const qf_gate *gates, size_t n_gates, uint32_t n, uint64_t batch, int sms);
int c128_seg_grid(int sms, uint64_t tiles);
cudaError_t launch_c128_prep(cudaStream_t st, int nsec, const uint32_t *off, const uint32_t *cnt,
                             const uint32_t *gates, const double *theta, double2 *secU);
// K: [section][3] (X, Y, Z); kpart: [grid][kC128MaxSec][3]
cudaError_t launch_c128_segment(cudaStream_t st, bool backward, int grid, const C128Seg &sg,
                                const C128Op *ops, const C128Round *rounds, const uint32_t *cz,
                                const double2 *secU, double2 *psi, double2 *lam, int n, uint32_t batch,
                                double *kpart, unsigned *ticket, double *K);
cudaError_t launch_c128_finalize(cudaStream_t st, int nsec, const uint32_t *off, const uint32_t *cnt,
                                 const uint32_t *gates, const double *theta, const double2 *secU,
                                 const double *K, double *grad);

// cudaFuncSetAttribute opt-ins (e.g. > 48 KiB of dynamic shared memory) are
// per device: `set` runs once on every device the process launches on (bit d
// of `done` = device d done). Racing first calls on one device both run `set`,
// which is idempotent.
template <class F> cudaError_t once_per_device(std::atomic<uint64_t> &done, F &&set) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (unsigned(dev) & 63u);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = set();
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

// Sets the thread-local qf_last_error() text (qf_capi.cpp).
void set_last_error(const char *msg);

} // namespace qfb
