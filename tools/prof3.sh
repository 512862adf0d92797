#!/bin/bash
# ncu --set full (source-level) of the steady-state backward A pass (hea20q, 20
# layers) and of the resident kernel (hea12q):  tools/prof3.sh TAG
set -u
TAG=$1; shift
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pass_bwd_dual \
  --launch-skip 7 -c 1 -o gpurun_out/prof_bwdA_${TAG} -f \
  python bench.py --steps 1 --warmup 0 --no-cpu --no-secondary --no-refsig --layers 20 "$@" \
  > gpurun_out/prof_bwdA_${TAG}.log 2>&1; echo "ncu bwdA rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:resident_kernel \
  --launch-skip 1 -c 1 -o gpurun_out/prof_res_${TAG} -f \
  python bench.py --workload hea12q --steps 1 --warmup 1 --no-cpu --no-secondary --no-refsig "$@" \
  > gpurun_out/prof_res_${TAG}.log 2>&1; echo "ncu res rc=$?"
