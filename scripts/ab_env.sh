#!/bin/bash
# A/B of an environment knob on the in-graph stamps: bash scripts/ab_env.sh VAR "v1 v2" "c1 c2 c3" rounds out
var=$1; vals=$2; confs=${3:-"c1 c2 c3"}; rounds=${4:-2}; out=${5:-gpurun_out/ab_env.txt}
for i in $(seq $rounds); do
  for v in $vals; do
    for c in $confs; do
      echo "== $var=$v $i $c" >> $out
      env $var=$v timeout 300 python scripts/timing_breakdown.py $c >> $out 2>&1
    done
  done
done
