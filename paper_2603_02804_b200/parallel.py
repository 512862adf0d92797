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
        self.inputs = None

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
        self.inputs = None  # device input buffers a plan may still be bound to

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


class HostInputPipeline:
    """End-to-end steps over a stream of host inputs with the next step's psi0
    H2D overlapped with the current step's gradient (double-buffered device
    copies, a copy stream; the plan reads them through qf_plan_set_psi0_device).
    Every step still copies its own inputs from pinned host memory and reads its
    [grad | loss] back; only the copy of step i+1 runs while step i computes."""

    def __init__(self, dp):
        torch = dp.torch
        self.dp = dp
        plan = dp.plan
        vals = plan.batch * (2 << plan.n)
        self.buf = [torch.empty(vals, dtype=torch.float32, device="cuda") for _ in range(2)]
        self.copy_stream = torch.cuda.Stream()
        self.copied = [torch.cuda.Event(), torch.cuda.Event()]
        self.done = [torch.cuda.Event(), torch.cuda.Event()]
        self.used = [False, False]

    def _issue_copy(self, slot, psi0_pinned):
        torch = self.dp.torch
        with torch.cuda.stream(self.copy_stream):
            if self.used[slot]:  # the step that last read this buffer has finished
                self.copy_stream.wait_event(self.done[slot])
            self.buf[slot].copy_(psi0_pinned, non_blocking=True)
            self.copied[slot].record(self.copy_stream)

    def run(self, psi0_list, theta_host_pinned, theta_dev, result_host):
        """Steps i = 0..len-1 on psi0_list[i] (pinned float32, batch * 2^(n+1)
        values each); result_host (pinned float64, M + 1) holds the last step's
        [grad | loss] once the plan stream is synchronized."""
        dp, torch = self.dp, self.dp.torch
        if not psi0_list:
            return result_host
        self._issue_copy(0, psi0_list[0])
        for i in range(len(psi0_list)):
            slot = i % 2
            if i + 1 < len(psi0_list):
                self._issue_copy(1 - slot, psi0_list[i + 1])
            with torch.cuda.stream(dp.stream):
                dp.stream.wait_event(self.copied[slot])
                dp.plan.set_psi0_device(self.buf[slot].data_ptr())
                theta_dev.copy_(theta_host_pinned, non_blocking=True)
                dp.step_device(theta_dev)
                result_host.copy_(dp.out[: dp.m + 1], non_blocking=True)
                self.done[slot].record(dp.stream)
                self.used[slot] = True
        return result_host

    def close(self):
        self.copy_stream.synchronize()
        self.buf = []


def combine_partials(partials):
    """Reference combine for tests: sum of per-rank (loss, grad) in rank order."""
    loss = sum(p[0] for p in partials)
    grad = np.sum([p[1] for p in partials], axis=0)
    return loss, grad
