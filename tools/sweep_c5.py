#!/usr/bin/env python
"""BASELINE config 5: qubit sweep n = 4..22 at a fixed 100 HEA layers, the
fused schedule against the per-gate (unfused) comparator, on one B200.

For every n, one JSON line:
  fused_hbm  samples/s of the fused gradient with the batch sized to HBM
             (B = 0.9 * free HBM / device bytes per sample, capped at 2^22
             samples), the config's own batch rule;
  fused/pergate at a common bounded batch (state = max(256 MiB, one tile
             group), > L2 for n >= 15) so the per-gate arm finishes in seconds:
             samples/s of both and their ratio, plus the per-gate algorithmic
             bytes (one traversal per gate: fwd 2S, bwd 4S per gate).
Timing: CUDA events inside the library (qf_stats.device_ms: theta H2D, all
kernels, [grad|loss|expect] D2H), one warm-up call, then the mean of --steps.
The checkpoint interval is k = 10 for n > 12 (sample-resident plans keep
their slots on chip).

    python tools/sweep_c5.py [--nmin 4 --nmax 22 --layers 100 --steps 2] > sweep.jsonl
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(plan, theta, steps, pergate=False):
    plan.gradient(theta, pergate=pergate)  # warm-up
    ms = [plan.gradient(theta, pergate=pergate).stats["device_ms"] for _ in range(steps)]
    return sum(ms) / len(ms)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nmin", type=int, default=4)
    ap.add_argument("--nmax", type=int, default=22)
    ap.add_argument("--layers", type=int, default=100)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--pergate-state-mib", type=int, default=256)
    ap.add_argument("--no-pergate", action="store_true")
    args = ap.parse_args()

    import torch
    import paper_2603_02804_b200 as pkg
    from paper_2603_02804_b200 import circuits as C

    ctx = pkg.Context(0)
    L = args.layers
    for n in range(args.nmin, args.nmax + 1):
        gates, M = C.build_hea(n, L)
        pauli = C.parse_pauli(C.repeated_ixyz_label(n))
        theta = C.random_parameters(M, 1235)
        k = 10
        S = 8 << n
        # device bytes per sample from two small plans
        db = []
        for b in (8, 16):
            p = pkg.Plan(ctx, gates, n, M, L, k, b, pauli)
            p.random_psi0(1234)
            db.append(p.gradient(theta).stats["device_bytes"])
            p.close()
        per_sample = max(1.0, (db[1] - db[0]) / 8.0)
        torch.cuda.empty_cache()
        free, _ = torch.cuda.mem_get_info()
        B = int(min(0.9 * (free - db[0]) / per_sample, 1 << 22))
        B = max(8, B - B % 8)
        line = {"n": n, "layers": L, "params": M, "ckpt_layers": k,
                "device_bytes_per_sample": per_sample}
        plan = pkg.Plan(ctx, gates, n, M, L, k, B, pauli)
        plan.random_psi0(1234)
        ms = timed(plan, theta, args.steps)
        st = plan.gradient(theta).stats
        line.update({"batch_hbm": B, "fused_hbm_ms": ms, "fused_hbm_sps": B / ms * 1e3,
                     "fused_hbm_GBps": st["hbm_bytes"] / ms / 1e6,
                     "fused_passes": st["forward_passes"] + st["backward_passes"],
                     "resident": st["resident"]})
        plan.close()
        torch.cuda.empty_cache()
        if not args.no_pergate:
            Bp = max(1, min(B, (args.pergate_state_mib << 20) // S))
            plan = pkg.Plan(ctx, gates, n, M, L, k, Bp, pauli)
            plan.random_psi0(1234)
            fms = timed(plan, theta, args.steps)
            pms = timed(plan, theta, max(1, args.steps // 2), pergate=True)
            ng = len(gates)
            pg_bytes = 6.0 * ng * Bp * S  # fwd 2S + bwd 4S per gate
            line.update({"batch_cmp": Bp, "fused_cmp_sps": Bp / fms * 1e3,
                         "pergate_cmp_sps": Bp / pms * 1e3, "fused_over_pergate": pms / fms,
                         "pergate_gates": ng, "pergate_GBps": pg_bytes / pms / 1e6})
            plan.close()
            torch.cuda.empty_cache()
        print(json.dumps(line), flush=True)
    os._exit(0)


if __name__ == "__main__":
    main()
