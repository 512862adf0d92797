#!/bin/bash
# ncu --set full of one steady-state balanced backward pass (kProgAlt) of hea20q
set -u
TAG=$1; shift
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pass_bwd_dual \
  --launch-skip 10 -c 1 -o gpurun_out/prof_alt_${TAG} -f \
  python bench.py --steps 1 --warmup 0 --no-cpu --no-secondary --no-refsig --layers 20 "$@" \
  > gpurun_out/prof_alt_${TAG}.log 2>&1; echo "ncu alt rc=$?"
