#!/bin/bash
# time the headline configurations (one line each) -> stdout
for c in "u16 7 gauss clamp" "u16 5 box clamp" "u16 3 gauss clamp" "f32 3 gauss clamp" "f32 5 box clamp" "f32 7 gauss clamp" "u8 3 gauss clamp" "u8 5 gauss clamp" "f32 3 lap wrap" "f32 5 box mirror"; do
  set -- $c
  timeout 60 python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --reps 5 2>&1 | tail -1
done
