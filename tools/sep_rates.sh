#!/bin/bash
# Separable vs dense tiled kernel rates at 1024^3 (CUDA events, best of 7).
for c in "u8 3 gauss clamp" "u16 3 gauss clamp" "u8 5 gauss clamp" "u16 7 gauss clamp" "f32 5 box clamp" \
         "f32 7 gauss clamp" "u16 9 gauss clamp" "f32 9 gauss clamp" "u16 7 gauss wrap" "u8 3 gauss mirror" "u16 7 gauss border"; do
  set -- $c
  for path in auto dense; do
    timeout 120 python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --n 1024 --reps 7 --path $path 2>&1 | tail -1
  done
done
