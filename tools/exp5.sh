python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edges.py tests/test_gpu_shard.py -q -p no:cacheprovider > gpurun_out/exp5_tests.log 2>&1
echo rc=$? >> gpurun_out/exp5_tests.log
VKT_LIB=build/sb/libvkt_b200.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edges.py -q -p no:cacheprovider > gpurun_out/exp5_tests_sb.log 2>&1
echo rc=$? >> gpurun_out/exp5_tests_sb.log
for lib in paper_2203_10213_b200/libvkt_b200.so build/sb/libvkt_b200.so; do
  for c in "u8 3 gauss clamp 1024" "u16 3 gauss clamp 1024" "u8 3 gauss clamp 256" "u8 3 gauss wrap 1024" "u16 3 gauss mirror 512" "u8 3 gauss border 512" "u16 3 box wrap 512"; do
    set -- $c
    VKT_LIB=$lib python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --n $5 --reps 7 2>&1 | sed "s|^|[$lib] |"
  done
done > gpurun_out/exp5.log 2>&1
bash tools/ncu_cases.sh r02d "u8 3 gauss clamp 1024"
