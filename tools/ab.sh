#!/bin/bash
# A/B timing of two builds of the library on the GPU box (interleaved runs).
#   tools/ab.sh LIB_A LIB_B [rounds] [bench args...]
A=$1; B=$2; R=${3:-2}; shift 3
for r in $(seq $R); do
  for L in $A $B; do
    QFUSE_B200_LIB=$L timeout 300 python bench.py --no-cpu --no-secondary --no-refsig "$@" 2>/dev/null | python3 -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1])
print('$L', round(d['value'],2), {k: round(v['ms'],1) for k,v in d['roofline']['per_kind'].items()})"
  done
done
