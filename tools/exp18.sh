VKT_WS=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edges.py -q -p no:cacheprovider -x > gpurun_out/exp18_tests.log 2>&1
echo rc=$? >> gpurun_out/exp18_tests.log
for env in "VKT_WS=1" "VKT_X=0"; do
  for c in "u8 3 gauss clamp 1024" "u16 3 gauss clamp 1024" "u8 3 gauss clamp 256" "u8 3 gauss wrap 1024" "u16 3 gauss mirror 512"; do
    set -- $c
    env $env timeout 120 python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --n $5 --reps 9 2>&1 | sed "s|^|[$env] |"
  done
done > gpurun_out/exp18.log 2>&1
VKT_WS=1 timeout 300 bash tools/ncu_cases.sh r02g "u8 3 gauss clamp 1024"
