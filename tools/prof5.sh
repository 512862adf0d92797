#!/bin/bash
# ncu --set full of one steady-state forward pass of each layout (hea20q, 20 layers)
set -u
TAG=$1; shift
mkdir -p gpurun_out
for K in wide:pass_fwd_wide narrow:pass_kernel; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${K#*:} \
  --launch-skip 6 -c 1 -o gpurun_out/prof_fwd_${K%%:*}_${TAG} -f \
  python bench.py --steps 1 --warmup 0 --no-cpu --no-secondary --no-refsig --layers 20 "$@" \
  > gpurun_out/prof_fwd_${K%%:*}_${TAG}.log 2>&1; echo "ncu ${K%%:*} rc=$?"
done
