#!/bin/bash
# chunk-depth sweep of the tiled kernel (VKT_TMA_ZC override)
for zc in 32 64 96 128 192 256 512; do
  echo -n "zc=$zc  "; VKT_TMA_ZC=$zc timeout 60 python tools/profile_case.py --fmt ${1:-u16} --k ${2:-7} --reps 4 2>&1 | tail -1
done
echo -n "auto   "; timeout 60 python tools/profile_case.py --fmt ${1:-u16} --k ${2:-7} --reps 4 2>&1 | tail -1
