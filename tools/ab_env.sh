#!/bin/bash
# A/B timing of environment-switched variants of the same build (interleaved):
#   tools/ab_env.sh "QF_WIDE=0" "QF_WIDE=1" [rounds] [bench args...]
A=$1; B=$2; R=${3:-2}; shift 3
for r in $(seq $R); do
  for V in "$A" "$B"; do
    env $V timeout 300 python bench.py --no-cpu --no-secondary --no-refsig "$@" 2>/dev/null | python3 -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1])
print('$V', round(d['value'],2), {k: round(v['ms']/v['launches']*1000,1) for k,v in d['roofline']['per_kind'].items()})"
  done
done
