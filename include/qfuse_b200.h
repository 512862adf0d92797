/* qfuse-b200 — C-ABI of the B200-native fused forward + adjoint-gradient
 * engine for batched state-vector circuits (arXiv 2603.02804).
 *
 * This is the drop-in boundary for the reference's hot path. The reference
 * (qfuse, /root/reference/proj) exposes it as C++ templates; each entry point
 * below replaces one of them (file:line under proj/):
 *
 *   qf_gradient_c64          <- qfuse::gradient<float>          include/qfuse/engine.hpp:139-142
 *                               qfuse::run_checkpointed<float>  include/qfuse/checkpoint.hpp:65-69
 *   qf_gradient_pergate_c64  <- qfuse::naive_gradient<float>    include/qfuse/engine.hpp:146-149
 *                               qfuse::run_checkpointed_naive   include/qfuse/checkpoint.hpp:73-79
 *   qf_plan_*                <- the same two calls with the circuit planned once and the
 *                               batch state resident in HBM (a training loop calls
 *                               gradient() with new theta every step, bench.cpp:114-133)
 *   qf_last_error            <- the what() of the exception the reference would throw
 *
 * Conventions (identical to the reference):
 *   - states are complex64, interleaved (re, im), sample-major: component (s, x)
 *     at s*2^(n+1) + 2x (+1)  (statevec.hpp:74-76); qubit t = bit t of x.
 *   - gates are the flattened IR (fusion.cpp:103-125): rotations u = cos(t/2) I
 *     - i sin(t/2) P (circuit.cpp:61-73), CZ, CNOT(control=q0, target=q1); every
 *     parameter slot is used by exactly one rotation (circuit.cpp:52-58).
 *   - observable: Pauli string masks (x_mask, z_mask) with Y = iXZ
 *     (circuit.hpp:98-108); y_count is recomputed as popcount(x & z).
 *   - loss = sum over samples of <psi_s|O|psi_s>; grad[j] = d loss / d theta_j,
 *     summed over the batch, fp64 (engine.cpp:733-738, :686-689).
 *
 * Return codes: 0 ok, 2 invalid argument (std::invalid_argument in the
 * reference), 3 capacity (qfuse::CapacityError), 4 CUDA/NCCL/internal
 * (std::logic_error / runtime failures). No exception crosses the ABI.
 * The caller owns host buffers; the library owns device memory. One context
 * per device; calls on one context are serialised by the caller.
 */
#ifndef QFUSE_B200_H
#define QFUSE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QF_OK 0
#define QF_EINVAL 2
#define QF_ECAPACITY 3
#define QF_EDEVICE 4

enum { QF_GATE_ROTATION = 0, QF_GATE_CZ = 1, QF_GATE_CNOT = 2 };
/* qfuse::StorageMode (engine.hpp:30). MEMSAVE keeps the checkpoint slots as
 * bfloat16 (narrow_to_bf16, statevec.hpp:36-45; half the slot memory); compute
 * and the final state stay complex64. The reference narrows its per-op ledger
 * instead (engine.cpp:488-513); both are held to the same tolerance (5e-3 of
 * the fp32 gradient, acceptance.cpp:466-499). Sample-resident plans (n <= 12)
 * store nothing per layer off-chip and run MEMSAVE at full precision. */
#define QF_STORAGE_FULL 0
#define QF_STORAGE_MEMSAVE 1
enum { QF_AXIS_X = 0, QF_AXIS_Y = 1, QF_AXIS_Z = 2 };

/* One flattened gate (qfuse::Gate, circuit.hpp:28-49). 16 bytes. */
typedef struct qf_gate {
    uint8_t kind;  /* QF_GATE_* */
    uint8_t axis;  /* QF_AXIS_* (rotations) */
    uint16_t pad;
    uint32_t q0;   /* rotation target, or control */
    uint32_t q1;   /* target of CZ/CNOT */
    uint32_t param;/* rotation parameter slot */
} qf_gate;

/* Mirrors qfuse::RunStats (engine.hpp:54-63) with device-side additions. */
typedef struct qf_stats {
    uint64_t forward_passes;     /* fused HBM passes in the forward (incl. replay) */
    uint64_t backward_passes;    /* fused HBM passes in the backward */
    uint64_t observable_passes;  /* expectation + adjoint seed passes */
    uint64_t kernel_launches;    /* kernels launched by this call */
    uint64_t hbm_bytes;          /* algorithmic HBM bytes moved by the fused passes */
    uint64_t device_bytes;       /* device memory held by the plan */
    uint32_t passes_per_layer;   /* P */
    uint32_t ckpt_layers;        /* k actually used */
    uint32_t resident;           /* 1 if one sample group stays in shared memory */
    uint32_t stages;             /* device stages (= layers for HEA) */
    double device_ms;            /* CUDA-event time of the device work */
} qf_stats;

typedef struct qf_ctx qf_ctx;
typedef struct qf_plan qf_plan;

const char *qf_last_error(void);
const char *qf_version(void);

int qf_ctx_create(int device, qf_ctx **out);
int qf_ctx_destroy(qf_ctx *ctx);
/* Optional HBM budget (bytes) checked before allocation; 0 = free memory. */
int qf_ctx_set_hbm_limit(qf_ctx *ctx, uint64_t bytes);
/* One-shot calls (qf_gradient_c64, _ex, _pergate_c64) keep their plan in the
 * context and reuse it while the next call has the same gates, shape and
 * storage mode (a training loop: the reference's gradient<float> called with new
 * theta and psi0 every step, bench.cpp:114-133); the host psi0 is staged through
 * a pinned buffer by host threads, overlapped with the DMA. Creating a plan on
 * the context drops the cached one first. enable = 0 turns the cache off and
 * frees the cached plan and the staging buffer. Default on. */
int qf_ctx_set_plan_cache(qf_ctx *ctx, int enable);

/* One-shot fused forward + adjoint gradient (the reference's
 * gradient<float> / run_checkpointed<float>). layers: number of equal
 * layer periods in the gate list (CheckpointPlan::uniform, checkpoint.cpp:38-49);
 * ckpt_layers: checkpoint interval k in layers, 0 = engine default; must
 * divide layers. psi0: host, batch*2^(n+1) floats. grad_out: n_params doubles.
 * expect_out (nullable): per-sample <O>. stats_out nullable. */
int qf_gradient_c64(qf_ctx *ctx, const qf_gate *gates, size_t n_gates, uint32_t n_qubits,
                    uint32_t n_params, uint32_t layers, uint32_t ckpt_layers,
                    const float *psi0, uint32_t batch, const double *theta,
                    uint64_t x_mask, uint64_t z_mask, double *loss_out, double *grad_out,
                    double *expect_out, qf_stats *stats_out);

/* Same with the reference's StorageMode (QF_STORAGE_*). */
int qf_gradient_c64_ex(qf_ctx *ctx, const qf_gate *gates, size_t n_gates, uint32_t n_qubits,
                       uint32_t n_params, uint32_t layers, uint32_t ckpt_layers,
                       uint32_t storage_mode, const float *psi0, uint32_t batch,
                       const double *theta, uint64_t x_mask, uint64_t z_mask, double *loss_out,
                       double *grad_out, double *expect_out, qf_stats *stats_out);
/* Per-gate (unfused) comparator: one HBM traversal per gate, the
 * reference's naive_gradient (engine.cpp:856-894). Same arguments. */
int qf_gradient_pergate_c64(qf_ctx *ctx, const qf_gate *gates, size_t n_gates,
                            uint32_t n_qubits, uint32_t n_params, uint32_t layers,
                            uint32_t ckpt_layers, const float *psi0, uint32_t batch,
                            const double *theta, uint64_t x_mask, uint64_t z_mask,
                            double *loss_out, double *grad_out, double *expect_out,
                            qf_stats *stats_out);

/* Forward only (the reference's forward<float>, engine.hpp:131-133): the final
 * state psi_M before the observable, batch*2^(n+1) floats to host, global phase
 * included (amplitude for amplitude the reference's). One-shot like
 * qf_gradient_c64 (plan cached in the context). */
int qf_forward_c64(qf_ctx *ctx, const qf_gate *gates, size_t n_gates, uint32_t n_qubits,
                   uint32_t n_params, uint32_t layers, const float *psi0, uint32_t batch,
                   const double *theta, float *psi_out, qf_stats *stats_out);

/* complex128 (the reference's double instantiations, engine.cpp:942,
 * checkpoint.cpp:196-213): psi0 is batch*2^(n+1) doubles. Fused fp64 segments:
 * each HBM pass applies every op whose target fits one 1024-amplitude tile
 * (sections of consecutive rotations as one 2x2 unitary, CZ runs, CNOTs),
 * psi uncomputed in place (ckpt_layers is validated, not needed).
 * Same arguments and errors as qf_gradient_c64. */
int qf_gradient_c128(qf_ctx *ctx, const qf_gate *gates, size_t n_gates, uint32_t n_qubits,
                     uint32_t n_params, uint32_t layers, uint32_t ckpt_layers,
                     const double *psi0, uint32_t batch, const double *theta,
                     uint64_t x_mask, uint64_t z_mask, double *loss_out, double *grad_out,
                     double *expect_out, qf_stats *stats_out);
/* complex128 per-gate schedule (one HBM traversal per gate): the reference's
 * naive_gradient<double> / run_checkpointed_naive<double> (engine.cpp:856-894,
 * checkpoint.cpp:165-188). Same arguments as qf_gradient_c128. */
int qf_gradient_pergate_c128(qf_ctx *ctx, const qf_gate *gates, size_t n_gates,
                             uint32_t n_qubits, uint32_t n_params, uint32_t layers,
                             uint32_t ckpt_layers, const double *psi0, uint32_t batch,
                             const double *theta, uint64_t x_mask, uint64_t z_mask,
                             double *loss_out, double *grad_out, double *expect_out,
                             qf_stats *stats_out);

/* ---- planned / HBM-resident interface (training loops, bench) ---- */

/* Plans the circuit once (theta-independent) and allocates the batch store,
 * checkpoint slots and scratch for `batch` samples on ctx's device. */
int qf_plan_create(qf_ctx *ctx, const qf_gate *gates, size_t n_gates, uint32_t n_qubits,
                   uint32_t n_params, uint32_t layers, uint32_t ckpt_layers, uint32_t batch,
                   uint64_t x_mask, uint64_t z_mask, qf_plan **out);
/* Same with the reference's StorageMode (QF_STORAGE_*). */
int qf_plan_create_ex(qf_ctx *ctx, const qf_gate *gates, size_t n_gates, uint32_t n_qubits,
                      uint32_t n_params, uint32_t layers, uint32_t ckpt_layers, uint32_t batch,
                      uint64_t x_mask, uint64_t z_mask, uint32_t storage_mode, qf_plan **out);
int qf_plan_destroy(qf_plan *plan);
/* Batch store input. Host (pageable or pinned) -> device copy. */
int qf_plan_upload_psi0(qf_plan *plan, const float *psi0_host);
/* Or point the plan at caller-owned device memory (batch*2^(n+1) floats on the
 * plan's device, 16-byte aligned; batch*2^n a multiple of 16): it is aliased,
 * not copied and never written, and stays bound until the next
 * qf_plan_upload_psi0 / qf_plan_random_psi0 (which go back to the plan's own
 * store). Every later gradient reads it on the plan's stream (qf_plan_stream):
 * the caller orders its writes to the buffer before those calls (same stream,
 * or an event the plan stream waits on) and keeps it alive while bound. */
int qf_plan_set_psi0_device(qf_plan *plan, const float *psi0_device);
/* Fused forward + adjoint gradient. theta/outputs are HOST pointers. */
int qf_plan_gradient(qf_plan *plan, const double *theta, double *loss_out, double *grad_out,
                     double *expect_out, qf_stats *stats_out);
/* Same, device pointers: theta_dev (n_params doubles, device); out_dev receives
 * [grad (n_params) | loss (1) | expect (batch)] doubles on the device. Enqueued on
 * the plan's stream; no host synchronisation. */
int qf_plan_gradient_device(qf_plan *plan, const double *theta_dev, double *out_dev);
/* Per-gate comparator on the same plan's store. */
int qf_plan_gradient_pergate(qf_plan *plan, const double *theta, double *loss_out,
                             double *grad_out, double *expect_out, qf_stats *stats_out);
/* Forward only: final state (before the observable) to host, complex64. */
int qf_plan_forward_state(qf_plan *plan, const double *theta, float *psi_out_host);
/* Stream the plan enqueues on (cudaStream_t as void*) and a sync helper. */
void *qf_plan_stream(qf_plan *plan);
int qf_plan_synchronize(qf_plan *plan);
/* Algorithmic HBM bytes of one fused gradient (schedule of this plan), and
 * the same split per pass kind, for roofline reporting. */
int qf_plan_traffic(const qf_plan *plan, uint64_t *total_bytes, uint64_t *pass_bytes,
                    uint64_t *passes_per_gradient);

/* Host-only description of the schedule qf_plan_create would build (no device, no
 * allocation): the planner's decisions, for tests and capacity planning. */
typedef struct qf_plan_info {
    uint32_t stages;           /* device stages (HEA: one per layer) */
    uint32_t resident;         /* 1: sample-resident kernel (n <= 12) */
    uint32_t layouts;          /* streaming pass layouts (0 when resident) */
    uint32_t passes;           /* forward passes per gradient (= backward passes) */
    uint32_t slots;            /* checkpoint slots */
    uint32_t ckpt_passes;      /* passes per checkpoint block */
    uint32_t balanced;         /* 1: balanced backward schedule (17 <= n <= 20, even block) */
    uint32_t wide_forward;     /* forward passes on the 64-amplitude wide kernel */
    uint32_t compiled_forward; /* forward passes on compiled phase programs (incl. wide) */
    uint32_t compiled_backward;/* backward passes on compiled phase programs */
    uint64_t bytes_per_sample; /* algorithmic HBM bytes of one gradient per sample
                                  (fwd 2S, bwd 4S or 3S after a slot, observable 2S;
                                  resident: psi0 + slot writes and reads) */
} qf_plan_info;
int qf_plan_describe(const qf_gate *gates, size_t n_gates, uint32_t n_qubits, uint32_t n_params,
                     uint32_t layers, uint32_t ckpt_layers, uint32_t batch, uint64_t x_mask,
                     uint64_t z_mask, qf_plan_info *out);

/* Synthetic batch store on the device: new_random_state<float>(n, batch, seed)
 * (statevec.cpp:32-53) for samples [first_sample, first_sample + batch) of
 * the global stream, written straight into the plan's psi0 store. */
int qf_plan_random_psi0(qf_plan *plan, uint64_t seed, uint64_t first_sample);
/* Copy the plan's psi0 store back to host memory (batch*2^(n+1) floats). */
int qf_plan_download_psi0(qf_plan *plan, float *psi0_host);

/* Per-launch CUDA-event profiling by kernel kind (for roofline reporting).
 * Kinds: 0 forward pass, 1 backward pass, 2 observable, 3 sample-resident,
 * 4 prep/reduce/finalize, 5 per-gate, 6 MemSave slot narrow/widen.
 * bytes = algorithmic HBM bytes. */
typedef struct qf_profile {
    uint64_t launches[8];
    double ms[8];
    double bytes[8];
} qf_profile;
int qf_plan_set_profiling(qf_plan *plan, int enable);
int qf_plan_profile(qf_plan *plan, qf_profile *out, int reset);
/* Counters of the plan's last gradient (qf_plan_gradient* / _device). */
int qf_plan_last_stats(const qf_plan *plan, qf_stats *out);

/* ---- multi-GPU, one process ----
 * Samples are independent and loss/gradient are sums over samples
 * (engine.cpp:733-738, :686-689): device i of the group owns the contiguous
 * sample range [i*B/G + min(i, B%G), ...) (sizes differ by at most one), runs
 * the whole fused gradient on its shard, and the only exchange is one
 * ncclAllReduce(sum, fp64) of [grad | loss] (n_params + 1 doubles) across the
 * group over NVLink. NCCL is loaded at qf_group_create (libnccl.so.2); if it
 * is missing the call fails with QF_EDEVICE. A multi-process job (one rank per
 * GPU, torchrun) uses qf_plan_gradient_device + its own all-reduce instead.
 * expect_out receives every sample's <O> in global order. stats_out sums the
 * counters over devices; device_ms is the max over devices. */
typedef struct qf_group qf_group;
typedef struct qf_group_plan qf_group_plan;
/* devices: n_gpus distinct CUDA ordinals, or NULL for 0..n_gpus-1. */
int qf_group_create(int n_gpus, const int *devices, qf_group **out);
int qf_group_destroy(qf_group *group);
int qf_group_size(const qf_group *group);
/* Plans the circuit once on every device for `batch` global samples. */
int qf_group_plan_create(qf_group *group, const qf_gate *gates, size_t n_gates,
                         uint32_t n_qubits, uint32_t n_params, uint32_t layers,
                         uint32_t ckpt_layers, uint32_t batch, uint64_t x_mask, uint64_t z_mask,
                         uint32_t storage_mode, qf_group_plan **out);
int qf_group_plan_destroy(qf_group_plan *gplan);
/* psi0_host: the whole batch (batch*2^(n+1) floats); each device copies its shard. */
int qf_group_plan_upload_psi0(qf_group_plan *gplan, const float *psi0_host);
/* new_random_state<float>(n, batch, seed) on the devices (global sample order). */
int qf_group_plan_random_psi0(qf_group_plan *gplan, uint64_t seed);
int qf_group_plan_gradient(qf_group_plan *gplan, const double *theta, double *loss_out,
                           double *grad_out, double *expect_out, qf_stats *stats_out);
/* The one-shot multi-GPU call (the reference's gradient<float> /
 * run_checkpointed<float> over n_gpus devices). The group for a device list is
 * created on first use and kept for the life of the process. */
int qf_gradient_c64_multi(int n_gpus, const int *devices, const qf_gate *gates, size_t n_gates,
                          uint32_t n_qubits, uint32_t n_params, uint32_t layers,
                          uint32_t ckpt_layers, uint32_t storage_mode, const float *psi0,
                          uint32_t batch, const double *theta, uint64_t x_mask, uint64_t z_mask,
                          double *loss_out, double *grad_out, double *expect_out,
                          qf_stats *stats_out);

#ifdef __cplusplus
}
#endif

#endif /* QFUSE_B200_H */
