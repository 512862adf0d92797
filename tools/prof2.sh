#!/bin/bash
# ncu --set full (source-level) of steady-state pass kernels (run under gpurun
# from the repo root):  tools/prof2.sh TAG [extra bench args]
# Captures 2 backward (layouts B, A) and 2 forward (A, B) launches of a 20-layer
# hea20q gradient; reports land in gpurun_out/prof_{bwd,fwd}_TAG.ncu-rep.
set -u
TAG=$1; shift
mkdir -p gpurun_out
for K in bwd:pass_bwd_dual fwd:pass_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${K#*:} \
    --launch-skip 6 -c 2 -o gpurun_out/prof_${K%%:*}_${TAG} -f \
    python bench.py --steps 1 --warmup 0 --no-cpu --no-secondary --no-refsig --layers 20 "$@" \
    > gpurun_out/prof_${K%%:*}_${TAG}.log 2>&1; echo "ncu ${K%%:*} rc=$?"
done
