#!/bin/bash
# ncu --set full captures of one filter_tma launch per case -> gpurun_out/<tag>_<case>.ncu-rep
# usage: bash tools/ncu_cases.sh TAG "u8 3 gauss clamp 1024" ["f32 5 box clamp 1024" ...]
tag=$1; shift
mkdir -p gpurun_out
for c in "$@"; do
  set -- $c
  name="${tag}_$1k$2$3_$4_$5"
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"filter_(tma|warp|ws|sep)" -c 1 \
    -o gpurun_out/$name -f python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --n $5 --reps 1 \
    > gpurun_out/$name.log 2>&1
done
