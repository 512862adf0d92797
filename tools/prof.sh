#!/bin/bash
# Profiling recipe used for profiles/ (run under gpurun from the repo root).
#   tools/prof.sh TAG [extra bench args]
# 1) launch list (serialised, cold-cache; shares only) on a 100-layer run
# 2) ncu --set full of one steady-state backward and one forward pass
set -u
TAG=$1; shift
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 1 --warmup 1 --no-cpu --layers 100 "$@" \
  > gpurun_out/launches_${TAG}.log 2>&1; echo "launch list rc=$?"
for K in bwd:pass_bwd_dual fwd:pass_kernel; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:${K#*:} \
    --launch-skip 6 -c 2 -o gpurun_out/prof_${K%%:*}_${TAG} -f \
    python bench.py --steps 1 --warmup 0 --no-cpu --layers 20 "$@" \
    > gpurun_out/prof_${K%%:*}_${TAG}.log 2>&1; echo "ncu ${K%%:*} rc=$?"
done
