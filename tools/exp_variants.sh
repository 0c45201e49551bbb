#!/bin/bash
# time the diagnostics builds under build/<variant>/ on one case
for v in product $(ls build | grep -v '^obj'); do
  lib=build/$v/libvkt_b200.so; [ $v = product ] && lib=paper_2203_10213_b200/libvkt_b200.so
  echo -n "$v: "; VKT_LIB=$lib timeout 60 python tools/profile_case.py "$@" --reps 4 2>&1 | tail -1 | sed 's/(all.*//'
done
