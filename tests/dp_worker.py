"""Worker of tests/test_gpu_multi.py::test_data_parallel_gradient_world2 (run by
torch.distributed.run, one process per rank; all ranks may share cuda:0).

Each rank plans its contiguous shard of the batch, generates its slice of the
global SplitMix64 stream on the device, and runs DataParallelGradient.step_device
(fused gradient + all-reduce of [grad | loss] over the process group, the
product path of bench.py). Rank 0 also runs the whole batch on one plan and
writes both results to $QF_DP_OUT.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2603_02804_b200 as pkg  # noqa: E402
from paper_2603_02804_b200 import circuits as C  # noqa: E402
from paper_2603_02804_b200.parallel import DataParallelGradient, shard_range  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist.init_process_group(os.environ.get("QF_DIST_BACKEND", "gloo"))
    n, layers, k, batch = int(os.environ.get("QF_DP_N", "14")), 4, 2, 7
    gates, M = C.build_hea(n, layers)
    pauli = C.parse_pauli(C.repeated_ixyz_label(n))
    theta = C.random_parameters(M, 1235)
    a, b = shard_range(batch, rank, world)
    ctx = pkg.Context(dev)
    plan = pkg.Plan(ctx, gates, n, M, layers, k, b - a, pauli)
    plan.random_psi0(1234, first_sample=a)
    dp = DataParallelGradient(plan, torch, dist)
    theta_d = torch.from_numpy(theta).cuda()
    out = dp.step_device(theta_d)
    dp.stream.synchronize()
    red = out[: M + 1].cpu().numpy().copy()
    exp_local = out[M + 1:].cpu().numpy().copy()
    # per-sample expectations gathered in rank order
    parts = [None] * world
    dist.all_gather_object(parts, exp_local.tolist())
    if rank == 0:
        full_plan = pkg.Plan(ctx, gates, n, M, layers, k, batch, pauli)
        full_plan.random_psi0(1234)
        single = full_plan.gradient(theta)
        np.savez(os.environ["QF_DP_OUT"], red=red, expect=np.concatenate(parts),
                 single_grad=single.gradient, single_loss=single.loss,
                 single_expect=single.expect)
        full_plan.close()
    dp.close()
    plan.close()
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
