#!/bin/bash
# the cfg5 filter (512^3 u8 Gaussian 5^3) and cfg2 (512^3 f32 box 5^3) under every address mode
for m in wrap mirror clamp border; do
  timeout 60 python tools/profile_case.py --fmt u8 --k 5 --n 512 --mode $m --reps 8 2>&1 | tail -1 | sed 's/(all.*//'
done
for m in wrap mirror clamp border; do
  timeout 60 python tools/profile_case.py --fmt f32 --k 5 --kernel box --n 512 --mode $m --reps 8 2>&1 | tail -1 | sed 's/(all.*//'
done
