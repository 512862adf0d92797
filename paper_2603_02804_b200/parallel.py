"""Batch-sharded data parallelism over the GPUs of one box.

Samples are independent and loss/gradient are sums over samples
(engine.cpp:733-738, :686-689), so rank r owns the contiguous sample range
shard_range(B, r, G) of the global stream and the only exchange is one
all-reduce(sum, fp64) of [grad (M) | loss] per step over NCCL/NVLink
(SURVEY §8e). No data-path collective exists besides that reduction.
"""
from __future__ import annotations

import numpy as np


def shard_range(batch: int, rank: int, world: int):
    """Contiguous [start, stop) of rank's samples; sizes differ by at most one."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


class DataParallelGradient:
    """One rank's share of a data-parallel gradient step.

    ``plan`` is this rank's capi.Plan over its shard; ``out`` a CUDA float64
    tensor of plan.n_params + 1 + plan.batch entries. gradient_device() enqueues
    the fused gradient on the plan's stream and all-reduces [grad | loss] on the
    same stream, so the caller sees the global sums in out[:M+1].
    """

    def __init__(self, plan, torch_mod, dist_mod=None):
        self.plan = plan
        self.torch = torch_mod
        self.dist = dist_mod
        self.stream = torch_mod.cuda.ExternalStream(plan.stream())
        m = plan.n_params
        self.out = torch_mod.empty(m + 1 + plan.batch, dtype=torch_mod.float64, device="cuda")
        self.m = m

    def step_device(self, theta_dev):
        torch = self.torch
        with torch.cuda.stream(self.stream):
            self.plan.gradient_device(theta_dev.data_ptr(), self.out.data_ptr())
            if self.dist is not None and self.dist.is_initialized() and self.dist.get_world_size() > 1:
                self.dist.all_reduce(self.out[: self.m + 1])
        return self.out

    def close(self):
        """Waits for this rank's queued work and drops the device buffers, so the
        plan and its context (which own the stream) can be destroyed next."""
        if self.out is not None:
            self.stream.synchronize()
            self.out = None

    def step_host(self, psi0_pinned, theta_host_pinned, theta_dev, result_host):
        """End-to-end step with host buffers: H2D psi0 + theta, gradient,
        all-reduce, D2H [grad | loss]. Returns result_host (pinned float64)."""
        torch = self.torch
        with torch.cuda.stream(self.stream):
            self.plan.upload_psi0_ptr(psi0_pinned.data_ptr())
            theta_dev.copy_(theta_host_pinned, non_blocking=True)
            self.step_device(theta_dev)
            result_host.copy_(self.out[: self.m + 1], non_blocking=True)
        return result_host


def combine_partials(partials):
    """Reference combine for tests: sum of per-rank (loss, grad) in rank order."""
    loss = sum(p[0] for p in partials)
    grad = np.sum([p[1] for p in partials], axis=0)
    return loss, grad
