#!/bin/bash
# chunk-depth sweep: bash tools/zc_sweep2.sh "<profile_case args>" z1 z2 ...
args=$1; shift
for z in auto "$@"; do
  if [ $z = auto ]; then unset VKT_TMA_ZC; else export VKT_TMA_ZC=$z; fi
  echo -n "zc=$z: "; timeout 60 python tools/profile_case.py $args --reps 8 2>&1 | tail -1 | sed 's/(all.*//'
done
