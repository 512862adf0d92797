#!/usr/bin/env python
"""Benchmark: samples/s of the fused forward + full adjoint gradient of a
batched 20-qubit HEA (BASELINE.json metric), with HBM roofline, end-to-end
leg, clocks and the reference's CPU implementation timed on the host.

    python bench.py [--gpus N --steps K --warmup W] [--workload hea20q]
    python bench.py --impl reference ...      # the reference (oracle/_ref), CPU

Workload (default ``hea20q``): BASELINE config 4's per-GPU shard — HEA 20
qubits x 1000 layers (60,000 params), 125 samples per GPU, checkpoint every
10 layers; weak scaling (N GPUs hold N x 125 samples; N = 8 is config 4's
1000 samples). A step = one fused forward + adjoint gradient over the rank's
samples plus the NCCL all-reduce of [grad | loss]. Inputs: ψ0 =
new_random_state<float>(20, N*125, 1234) (each rank its slice of the global
stream, generated on the device), θ = random_parameters(60000, 1235),
O = IXYZ.... The state (1 GiB per GPU) is larger than L2.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "samples/sec fwd+adjoint grad, 20q HEA; achieved HBM GB/s vs roofline"
WORKLOADS = {
    # name: qubits, layers, per-GPU batch, checkpoint layers, BASELINE config
    "hea20q": dict(n=20, layers=1000, batch=125, ckpt=10, config="configs[3] per-GPU shard"),
    "hea16q": dict(n=16, layers=200, batch=1024, ckpt=10, config="configs[2]"),
    "hea12q": dict(n=12, layers=100, batch=1024, ckpt=10, config="configs[1]"),
    "hea4q": dict(n=4, layers=4, batch=8, ckpt=0, config="configs[0]"),
}
SEED_STATE, SEED_THETA = 1234, 1235
FALLBACK_HBM_GBS = 6650.0


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.tmp = None

    def start(self):
        try:
            self.tmp = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.gpu)], stdout=self.tmp, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.tmp.flush()
        rows = []
        with open(self.tmp.name) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.tmp.name)
        if not rows:  # timed region shorter than nvidia-smi's start-up: one query right after
            try:
                out = subprocess.run(["nvidia-smi", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits", "-i", str(self.gpu)],
                                     capture_output=True, text=True, timeout=20).stdout
                rows = [[x.strip() for x in line.split(",")] for line in out.splitlines()
                        if len(line.split(",")) >= 9]
            except (OSError, subprocess.TimeoutExpired):
                rows = []
            if not rows:
                return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
            self.note = "sampled once right after the timed region (region shorter than the sampler start-up)"
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        power = [float(r[3]) for r in rows if r[3].replace(".", "").isdigit()]
        res = {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons,
               "samples": len(rows), "power_w_max": max(power) if power else None}
        if getattr(self, "note", None):
            res["note"] = self.note
        return res


# ------------------------------------------------------------ CPU legs
def reference_sample(ref, n, layers_total, threads, budget_s=12.0):
    """Time the reference's run_checkpointed<float> (oracle/_ref, OpenMP, all
    threads) on a bounded sample of the workload and extrapolate linearly in
    layers (CPU time is linear in B*d)."""
    import numpy as np
    from paper_2603_02804_b200 import circuits as C
    ref.set_threads(threads)
    batch = max(threads, 1)
    pauli = C.parse_pauli(C.repeated_ixyz_label(n))
    # probe one layer to size the sample
    layers = 1
    while True:
        gates, npar = C.build_hea(n, layers)
        theta = C.random_parameters(npar, SEED_THETA)
        psi0 = ref.random_state(n, batch, SEED_STATE, np.float32)
        t0 = time.perf_counter()
        ref.gradient(gates, n, npar, psi0, theta, pauli, layers=layers, block_layers=1)
        dt = time.perf_counter() - t0
        if dt * 2 > budget_s or layers * 2 > layers_total:
            break
        layers *= 2
    sps = batch / dt * (layers / layers_total)
    sample = (f"{n}q x {layers} layers x {batch} samples (run_checkpointed<float>, k=1) in "
              f"{dt:.2f} s on {threads} threads of {cpu_model()} (OpenMP); samples/s "
              f"extrapolated x{layers}/{layers_total} to the {layers_total}-layer workload")
    return sps, sample, (layers, batch, dt)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_threads():
    """All host cores this process may use (torchrun exports OMP_NUM_THREADS=1,
    which must not throttle the reference's OpenMP arm)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracles import RefLib
    wl = WORKLOADS[args.workload]
    ref = RefLib()
    threads = host_threads()
    vals = []
    sample = None
    for i in range(args.warmup + args.steps):
        v, sample, _ = reference_sample(ref, wl["n"], wl["layers"], threads)
        if i >= args.warmup:
            vals.append(v)
    value = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * wl["batch"] * args.gpus / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": workload_config(args, wl),
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": threads,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(args, wl):
    return {"workload": f"{args.workload}: HEA {wl['n']}q x {wl['layers']}L, "
                        f"{wl['batch']} samples/GPU ({wl['config']})",
            "qubits": wl["n"], "layers": wl["layers"], "params": 3 * wl["n"] * wl["layers"],
            "batch_per_gpu": wl["batch"], "global_batch": wl["batch"] * args.gpus,
            "ckpt_layers": wl["ckpt"], "observable": "IXYZ repeated",
            "storage": getattr(args, "storage", "full"),
            "l2": "inputs larger than L2 (state per GPU > 126 MB)" if wl["n"] >= 16
            else "state fits L2/smem (sample-resident)",
            "parallelism": f"dp{args.gpus}"}


# ------------------------------------------------------------ GPU arm
def fp32_peak():
    fp = os.path.join(ROOT, "profiles", "fp32_peak.json")
    return json.load(open(fp))["tfma_per_s"] if os.path.exists(fp) else 36.9


def roofline_of(prof, steps, n, layers, B, workload):
    """Roofline block of the dominant kernel kind of a timed region: algorithmic
    bytes (or lane-FMA) per launch / its average CUDA-event launch time."""
    peak, peak_src = measured_peaks()
    kinds = {k: v for k, v in prof.items() if v["launches"]}
    dom = max(kinds, key=lambda k: kinds[k]["ms"])
    d = kinds[dom]
    total_kernel_ms = sum(v["ms"] for v in kinds.values())
    per_kind = {k: {"launches": v["launches"], "ms": v["ms"],
                    "GBps": v["bytes"] / (v["ms"] / 1e3) / 1e9 if v["ms"] else None}
                for k, v in kinds.items()}
    if dom == "resident":
        # sample-resident (n <= 12): FP32 CUDA-core bound; per stage
        # and amplitude: forward 2n (Ry, one FFMA2 per output) + 8 (diagonal),
        # backward 4n (Ry on psi and lambda) + 6n (X, Y, Z per qubit) + 16 (diagonal)
        per_amp = (2 * n + 8) + (10 * n + 16)
        lane_fma = per_amp * B * (1 << n) * layers * steps
        ach = lane_fma / (d["ms"] / 1e3) / 1e12
        pk = fp32_peak()
        return {"bound": "fp32", "kernel": dom, "achieved": ach, "peak": pk, "unit": "TFMA/s",
                "frac": ach / pk, "traffic": None,
                "peak_source": "tools/ffma_probe.cu on this pool (profiles/fp32_peak.json)",
                "lane_fma_per_amp_stage": per_amp, "avg_launch_ms": d["ms"] / d["launches"],
                "share_of_step": d["ms"] / max(total_kernel_ms, 1e-9), "per_kind": per_kind,
                "hbm_GBps": d["bytes"] / (d["ms"] / 1e3) / 1e9}
    achieved = d["bytes"] / (d["ms"] / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(f"{workload}:{dom}")
    roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
            "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
            "peak_source": peak_src,
            "bytes_per_launch": d["bytes"] / d["launches"],
            "avg_launch_ms": d["ms"] / d["launches"],
            "share_of_step": d["ms"] / max(total_kernel_ms, 1e-9),
            "per_kind": per_kind,
            "algorithmic_bytes": "per state S = B*2^n*8; fwd pass 2S, bwd pass 4S (3S at a "
                                 "checkpoint block start), observable 2S"}
    # FP32 (CUDA-core) co-bound of the dominant pass kind: per
    # amplitude per stage forward 2n + 8, backward 4n (Ry on psi, lambda) + 4n
    # (X, Y; Z chained) + 16 (diagonal)
    per_amp = {"backward_pass": 8 * n + 16, "forward_pass": 2 * n + 8}.get(dom)
    if per_amp:
        stages_per_launch = layers / max(1, d["launches"] / max(1, steps))
        lane_fma = per_amp * B * (1 << n) * stages_per_launch
        ach = lane_fma / (d["ms"] / d["launches"] / 1e3) / 1e12
        pk = fp32_peak()
        roof["fp32"] = {"achieved": ach, "peak": pk, "unit": "TFMA/s", "frac": ach / pk,
                        "lane_fma_per_amp_stage": per_amp,
                        "peak_source": "tools/ffma_probe.cu on this pool (profiles/fp32_peak.json)"}
    return roof


def measure(pkg, C, torch, dist, dev, rank, world, wl, batch_global, steps, warmup, storage,
            scaling, e2e=False, refsig=False, clocks=False, workload="hea20q"):
    """One workload: plan this rank's shard, warm up, time `steps` fused
    gradients (+ the all-reduce) with CUDA events on the plan stream, max over
    ranks. Returns (line fields, plan, dp) -- the caller closes them."""
    import numpy as np
    from paper_2603_02804_b200.parallel import DataParallelGradient, HostInputPipeline, shard_range
    n, layers, k = wl["n"], wl["layers"], wl["ckpt"]
    a, b = shard_range(batch_global, rank, world)
    B = b - a
    gates, M = C.build_hea(n, layers)
    pauli = C.parse_pauli(C.repeated_ixyz_label(n))
    ctx = pkg.Context(dev)
    plan = pkg.Plan(ctx, gates, n, M, layers, k, B, pauli, storage=storage)
    plan.random_psi0(SEED_STATE, first_sample=a)
    theta_h = torch.from_numpy(C.random_parameters(M, SEED_THETA)).pin_memory()
    theta_d = theta_h.to(f"cuda:{dev}")
    dp = DataParallelGradient(plan, torch, dist if world > 1 else None)
    stream = dp.stream
    res = {}

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{dev}")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(warmup):
        dp.step_device(theta_d)
    stream.synchronize()
    launches_per_step = plan.gradient(theta_h.numpy()).stats["kernel_launches"]
    plan.set_profiling(True)
    plan.profile(reset=True)
    sampler = ClockSampler(dev) if (rank == 0 and clocks) else None
    barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        dp.step_device(theta_d)
    e1.record(stream)
    stream.synchronize()
    torch.cuda.synchronize()
    if sampler:
        res["clocks"] = sampler.stop()
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    prof = plan.profile(reset=True)
    plan.set_profiling(False)
    ms_per_step = ms / steps
    res.update({"value": batch_global / (ms_per_step / 1000.0), "ms_per_step": ms_per_step,
                "steps": steps, "warmup": warmup, "scaling": scaling,
                "gpu_launches": int(launches_per_step * steps)})
    out = dp.out[: M + 1].double().cpu().numpy()
    assert np.all(np.isfinite(out)), "non-finite gradient"
    res["roofline"] = roofline_of(prof, steps, n, layers, B, workload)
    if n > 12:
        # whole step against the BASELINE formula B_U = S(6Pd + d/k + 1), P = 2
        peak, _ = measured_peaks()
        P = 2
        kk = k or min(layers, 10)
        bu = (1 << n) * 8 * (6 * P * layers + layers / kk + 1) * B
        res["roofline"]["step_formula_frac"] = bu / (ms_per_step / 1e3) / (peak * 1e9)
        res["roofline"]["step_formula"] = ("B_U = S(6Pd + d/k + 1) with P=2 (BASELINE.md §2); "
                                           "the paired-stage schedule moves P=1")

    if e2e:
        # end-to-end: host buffers, psi0 H2D (pinned) + theta H2D + gradient +
        # all-reduce + D2H of [grad | loss] inside the timed region
        psi_h = torch.empty(B * (2 << n), dtype=torch.float32).pin_memory()
        plan.download_psi0_ptr(psi_h.data_ptr())
        res_h = torch.empty(M + 1, dtype=torch.float64).pin_memory()
        dp.step_host(psi_h, theta_h, theta_d, res_h)
        stream.synchronize()
        barrier()
        torch.cuda.synchronize()
        # e2e: every step copies its own psi0 + theta from pinned host memory and reads
        # [grad | loss] back; the psi0 copy of step i+1 overlaps step i (HostInputPipeline,
        # double-buffered device inputs); timed from before the first copy to after the
        # last D2H (host-synchronised wall clock, max over ranks)
        pipe = HostInputPipeline(dp)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        pipe.run([psi_h] * steps, theta_h, theta_d, res_h)
        stream.synchronize()
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1000.0) / steps
        pipe.copy_stream.synchronize()
        dp.inputs = pipe  # the plan stays bound to the pipeline's buffers: keep them alive with dp
        assert np.all(np.isfinite(res_h.numpy()))
        res["e2e"] = {"value": batch_global / (e2e_ms / 1000.0), "unit": "samples/s",
                      "h2d_bytes_per_step": int(psi_h.numel() * 4 + theta_h.numel() * 8),
                      "d2h_bytes_per_step": int(res_h.numel() * 8), "ms_per_step": e2e_ms,
                      "api": "parallel.HostInputPipeline: pinned psi0/theta H2D per step (next "
                             "step's copy overlapping this step), qf_plan_gradient_device, "
                             "all-reduce, D2H of [grad | loss]"}
        if refsig and world == 1:
            # the reference-signature call: one-shot qf_gradient_c64 on PAGEABLE host
            # buffers (what qfuse::b200::run_checkpointed / gradient<float> do per
            # call, bench.cpp:114-133); the plan is cached in the context after the
            # first call, psi0 staged through pinned memory by host threads
            psi_np = psi_h.numpy().reshape(B, 1 << n, 2).copy()
            th_np = theta_h.numpy().copy()
            dp.close()
            plan.close()
            dp = plan = None
            torch.cuda.empty_cache()
            one = pkg.gradient_c64(ctx, gates, n, M, layers, k, psi_np, th_np, pauli,
                                   storage=storage)  # builds + caches the plan
            t0 = time.perf_counter()
            for _ in range(steps):
                one = pkg.gradient_c64(ctx, gates, n, M, layers, k, psi_np, th_np, pauli,
                                       storage=storage)
            rs_ms = (time.perf_counter() - t0) * 1000.0 / steps
            assert np.isfinite(one.loss)
            res["e2e_refsig"] = {
                "value": batch_global / (rs_ms / 1000.0), "unit": "samples/s", "ms_per_step": rs_ms,
                "h2d_bytes_per_step": int(psi_np.nbytes + th_np.nbytes),
                "d2h_bytes_per_step": int((M + 1 + B) * 8),
                "timer": "host wall clock around each synchronous call",
                "api": "qf_gradient_c64_ex (one-shot C-ABI behind qfuse::b200::run_checkpointed), "
                       "pageable numpy psi0/theta in, loss/grad/expect out"}
    res["_n_per_rank"] = B
    return res, ctx, plan, dp


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2603_02804_b200 as pkg
    from paper_2603_02804_b200 import circuits as C

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"note: WORLD_SIZE={world} but --gpus={args.gpus}; using WORLD_SIZE")
        args.gpus = world
    dev = local % max(1, torch.cuda.device_count())  # tolerate fewer GPUs than ranks (tests)
    torch.cuda.set_device(dev)
    if world > 1:
        backend = os.environ.get("QF_DIST_BACKEND", "nccl")  # gloo: single-GPU test of this path
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    wl = dict(WORKLOADS[args.workload])
    if args.batch:
        wl["batch"] = args.batch
    if args.layers:
        wl["layers"] = args.layers
    if args.ckpt is not None:
        wl["ckpt"] = args.ckpt
    n, layers = wl["n"], wl["layers"]
    # weak: wl["batch"] samples per GPU; strong: wl["batch"] samples over all GPUs
    batch_global = wl["batch"] * world if args.scaling == "weak" else wl["batch"]
    res, ctx, plan, dp = measure(pkg, C, torch, dist, dev, rank, world, wl, batch_global,
                                 args.steps, args.warmup, args.storage, args.scaling,
                                 e2e=True, refsig=not args.no_refsig, clocks=True,
                                 workload=args.workload)
    B = res.pop("_n_per_rank")
    cfg = workload_config(args, wl)
    cfg["batch_per_gpu"] = B
    cfg["global_batch"] = batch_global
    line = {
        "metric": METRIC, "value": res["value"], "unit": "samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (device SplitMix64/Box-Muller states seed 1234, theta seed 1235)",
        "config": cfg, "clocks": res.get("clocks"), "e2e": res["e2e"],
        "gpu_launches": res["gpu_launches"], "roofline": res["roofline"],
    }
    if "e2e_refsig" in res:
        line["e2e_refsig"] = res["e2e_refsig"]
    for obj in (dp, plan, ctx):
        if obj is not None:
            obj.close()
    del dp, plan, ctx
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    # ---- secondary blocks: the other BASELINE configs on this box, each timed the
    # same way with its own roofline (config 2 and 3 at N = 1; config 3 strong-scaled
    # over the N GPUs of a scaling run)
    if not args.no_secondary and args.workload == "hea20q" and not args.batch and not args.layers:
        sec = {}
        plans = [("hea16q", "full", "strong")]
        if world == 1:
            plans += [("hea12q", "full", "strong"), ("hea20q", "memsave", "weak")]
        for name, storage, scaling in plans:
            w2 = dict(WORKLOADS[name])
            bg = w2["batch"] if scaling == "strong" else w2["batch"] * world
            st = args.steps if name != "hea20q" else max(3, min(args.steps, 5))
            try:
                r2, c2, p2, d2 = measure(pkg, C, torch, dist, dev, rank, world, w2, bg, st,
                                         max(3, args.warmup), storage, scaling, workload=name)
            except Exception as exc:  # report, never hide the headline
                sec[f"{name}_{storage}"] = {"error": str(exc)}
                continue
            for obj in (d2, p2, c2):
                if obj is not None:
                    obj.close()
            del d2, p2, c2
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
            per = r2.pop("_n_per_rank")
            r2["config"] = {"workload": f"{name}: HEA {w2['n']}q x {w2['layers']}L "
                                        f"({w2['config']}), {bg} samples over {world} GPU(s)",
                            "global_batch": bg, "batch_per_gpu": per, "ckpt_layers": w2["ckpt"],
                            "storage": storage}
            r2["unit"] = "samples/s"
            sec[f"{name}" + ("_memsave" if storage == "memsave" else "")] = r2
        line["secondary"] = sec

    # ---- CPU baseline: the reference on this host, rank 0 at N = 1 only
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            from oracles import RefLib
            ref = RefLib()
            th = host_threads()
            sps, sample, _ = reference_sample(ref, n, layers, th)
            line["cpu_baseline"] = {"value": sps, "unit": "samples/s", "cores": th,
                                    "kind": "reference", "sample": sample}
        except Exception as exc:  # the box may lack the prebuilt reference
            line["cpu_baseline"] = {"value": None, "unit": "samples/s", "cores": 0,
                                    "kind": "reference", "sample": f"unavailable: {exc}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    torch.cuda.synchronize()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="hea20q", choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=0, help="override per-GPU batch")
    ap.add_argument("--layers", type=int, default=0, help="override layer count")
    ap.add_argument("--ckpt", type=int, default=None, help="override checkpoint layers")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--storage", default="full", choices=["full", "memsave"],
                    help="StorageMode: memsave keeps checkpoint slots in bf16")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: --batch samples per GPU (config 4); strong: the workload's "
                         "batch split over the GPUs (config 3)")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the secondary workload blocks (hea16q, hea12q, memsave)")
    ap.add_argument("--no-refsig", action="store_true",
                    help="skip the reference-signature (one-shot C-ABI) e2e leg")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
