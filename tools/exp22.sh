VKT_WS5=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edges.py tests/test_gpu_shard.py -q -p no:cacheprovider -x 2>&1 | tail -2 > gpurun_out/exp22_tests.log
for env in "VKT_WS5=1" "VKT_X=0"; do
  for c in "u8 5 gauss clamp 1024" "u16 5 box clamp 1024" "f32 5 box clamp 1024" "u8 5 gauss clamp 512" "u8 5 gauss wrap 512" "f32 5 box mirror 512"; do
    set -- $c
    env $env timeout 120 python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --n $5 --reps 9 2>&1 | sed "s|^|[$env] |"
  done
done > gpurun_out/exp22.log 2>&1
