python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edges.py tests/test_gpu_shard.py tests/test_gpu_baseline_configs.py -q -p no:cacheprovider > gpurun_out/exp13_tests.log 2>&1
echo rc=$? >> gpurun_out/exp13_tests.log
for c in "u16 7 gauss clamp 1024" "f32 7 gauss clamp 1024" "u8 7 gauss clamp 1024" "u16 5 box clamp 1024" "u8 5 gauss clamp 1024" "f32 5 box clamp 1024" "u16 9 box clamp 512" "u16 7 gauss wrap 1024"; do
  set -- $c
  python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --n $5 --reps 7 2>&1
done > gpurun_out/exp13.log 2>&1
