#!/bin/bash
# A/B of two library builds over the three BASELINE workloads (interleaved):
#   tools/ab3.sh LIB_A LIB_B [rounds]
A=$1; B=$2; R=${3:-2}
for W in "--layers 200" "--workload hea16q" "--workload hea12q"; do
  bash tools/ab.sh $A $B $R $W | sed "s|^|$W |"
done
