#!/usr/bin/env python
"""complex128 timing: fused fp64 segments (qf_gradient_c128) against the fp64
per-gate schedule (qf_gradient_pergate_c128) on HEA circuits, one B200.
Times: device_ms = CUDA events around the kernels (psi0 already on the device);
wall = the whole one-shot call (allocation, psi0 H2D, D2H); after one warm-up.

    python tools/c128_bench.py [--n 16 20] [--layers 20] [--batch 8]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[12, 16, 20])
    ap.add_argument("--layers", type=int, default=20)
    ap.add_argument("--batch", type=int, default=8)
    args = ap.parse_args()
    import numpy as np
    import paper_2603_02804_b200 as pkg
    from paper_2603_02804_b200 import circuits as C
    ctx = pkg.Context(0)
    for n in args.n:
        gates, M = C.build_hea(n, args.layers)
        theta = C.random_parameters(M, 1235)
        psi0 = C.new_random_state(n, args.batch, 1234, np.float64)
        pauli = C.parse_pauli(C.repeated_ixyz_label(n))
        line = {"n": n, "layers": args.layers, "batch": args.batch}
        res = {}
        for name, pg in (("fused", False), ("pergate", True)):
            pkg.gradient_c128(ctx, gates, n, M, args.layers, 0, psi0, theta, pauli, pergate=pg)
            t0 = time.perf_counter()
            r = pkg.gradient_c128(ctx, gates, n, M, args.layers, 0, psi0, theta, pauli, pergate=pg)
            dt = time.perf_counter() - t0
            res[name] = r
            dms = r.stats["device_ms"]
            line[f"{name}_wall_s"] = dt
            line[f"{name}_device_ms"] = dms
            line[f"{name}_sps"] = args.batch / (dms / 1e3)
            line[f"{name}_GBps"] = r.stats["hbm_bytes"] / (dms / 1e3) / 1e9
            line[f"{name}_passes"] = r.stats["forward_passes"] + r.stats["backward_passes"]
        line["speedup"] = line["pergate_device_ms"] / line["fused_device_ms"]
        line["max_abs_grad_diff"] = float(np.max(np.abs(res["fused"].gradient - res["pergate"].gradient)))
        print(json.dumps(line), flush=True)
    os._exit(0)


if __name__ == "__main__":
    main()
