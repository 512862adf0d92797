// Internal structures shared by the host planner (qf_plan.cpp, qf_capi.cpp)
// and the sm_100a kernels (qf_kernels.cu). Not part of the C-ABI.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>

namespace qfb {

// ---------------------------------------------------------------- geometry
// One tile = 4096 amplitudes (32 KiB of complex64) held in shared memory as
// 256 rows x 16 amplitudes (128 B), TMA SWIZZLE_128B. Local index l (12 bits):
// bits 0..3 = column = global qubits 0..3; bits 4..11 = row = 8 global qubits
// (a contiguous block starting at the pass's row_start) or, for n <= 12, the
// remaining qubits and then sample bits.
constexpr int kTileBits = 12;
constexpr int kTileAmps = 1 << kTileBits;
constexpr int kTileBytes = kTileAmps * 8;
constexpr int kThreads = 256; // 8 warps; 16 amplitudes per thread per group phase
constexpr int kMaxQubits = 28;

// Encoded section gate: bits 0..1 kind (0 Rx, 1 Ry, 2 Rz, 3 fixed H), bits 2.. param.
constexpr uint32_t kSecH = 3u;

// Quadratic-form view of a set of CZ gates (the sign of a diagonal stage):
// sign(x) = (-1)^{Q(x)}, Q(x) = XOR_{p<q} A_pq x_p x_q.
struct CzSet {
    uint32_t adj[32];      // symmetric adjacency (bit p of adj[q] = A_pq)
    uint32_t adjlo[32];    // adj[q] restricted to bits < q
    uint32_t qcol;         // 16-bit mask: bit j = Q(j) for the 4 column qubits
    uint32_t pad[3];
    uint8_t rowinfo[256];  // pass-A rows: bit 4 = Q(r<<4), bits 0..3 = col mask of A*(r<<4)
};

// Per-launch parameters of a streaming pass (forward or backward).
struct PassParams {
    int n;             // qubits
    int stage;         // device stage (layer)
    int row_start;     // first global qubit of the 8 row bits (4 for pass A)
    int tiles;         // tiles in the launch
    int tile_lo_bits;  // tile bits between the column and the rows (row_start - 4)
    int tile_hi_bits;  // tile bits above the rows within a sample (n - row_start - 8)
    uint32_t rot_mask; // 12 local bits that carry an Ry this pass
    uint32_t meas_mask;// local bits whose K is accumulated (backward)
    int has_diag;      // pass A: stage diagonal D_s applied (fwd: first; bwd: last)
    int write_psi;     // backward: store psi (0 at a checkpoint block start)
    int qmap[12];      // local bit -> global qubit
    const float2 *ry;  // [n] (cos, sin) of beta/2 for this stage
    const float2 *tcol;// [16] diag table of this stage (column bits)
    const float2 *trow;// [256]
    const float2 *tt1; // [256] tile bits 12..19
    const float2 *tt2; // [256] tile bits 20..27
    const CzSet *cz;   // CZ set of this stage's diagonal (nullptr = none)
    double *kpart;     // backward: &kpart[0][stage][0][0], layout [grid][stages][n][8]
    long long kstride; // stages*n*8: distance between CTAs in kpart
};

// Parameters of the sample-resident kernel (n <= 12): the whole circuit runs
// on one tile of packed samples held in shared memory.
struct ResidentParams {
    int n;
    int stages;
    int ckpt;          // checkpoint interval in stages (re-anchor the uncompute)
    int tiles;
    uint32_t batch;
    uint64_t x_mask, z_mask;
    uint32_t y_count;
    const float2 *ry;  // [stages][n]
    const float2 *tcol, *trow; // [stages][16], [stages][256]
    const CzSet *czsets;       // distinct CZ sets
    const int *stage_cz;       // [stages] index into czsets or -1
    const double *wfinal;      // [n] final diagonal phases
    const CzSet *czfinal;      // final CZ set (nullptr = none)
    double *kpart;             // [stages][n][8][grid]
    double *expect;            // [batch]
    int forward_only;          // 1: forward then store the final state
};

struct SeedParams {
    int n;
    uint32_t batch;
    uint64_t x_mask, z_mask;
    uint32_t y_count;
    const double *wfinal;
    const CzSet *czfinal;
    const float2 *psi;
    float2 *lam;
    double *epart; // [batch][chunks]
};

// Kernel launchers (qf_kernels.cu).
cudaError_t launch_prep_sections(cudaStream_t st, int n_sec, const uint32_t *sec_q,
                                 const uint32_t *sec_stage, const uint32_t *sec_alpha_row,
                                 const uint32_t *sec_off, const uint32_t *sec_gates,
                                 const double *theta, int n, float2 *ry, double *wg,
                                 double *wa, double *sec_gamma);
cudaError_t launch_diag_tables(cudaStream_t st, int stages, int n, const double *wg,
                               const double *wa, float2 *tcol, float2 *trow, float2 *tt1,
                               float2 *tt2, double *wfinal);
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

} // namespace qfb
