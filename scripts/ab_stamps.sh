#!/bin/bash
# A/B of the in-graph per-kernel stamps: current library vs build/ab_old/libdynscreen.so,
# alternating, on the same box.  Usage: bash scripts/ab_stamps.sh "c1 c2 c3" rounds out.txt
confs=${1:-"c1 c2 c3"}; rounds=${2:-2}; out=${3:-gpurun_out/ab.txt}
for i in $(seq $rounds); do
  for lib in new old; do
    if [ $lib = old ]; then export DSCR_LIB=$PWD/build/ab_old/libdynscreen.so; else unset DSCR_LIB; fi
    for c in $confs; do
      echo "== $lib $i $c" >> $out
      timeout 300 python scripts/timing_breakdown.py $c >> $out 2>&1
    done
  done
done
unset DSCR_LIB
