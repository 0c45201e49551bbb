VKT_LIB=$PWD/build/y2c5/libvkt_b200.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -p no:cacheprovider > gpurun_out/exp17_tests.log 2>&1
echo rc=$? >> gpurun_out/exp17_tests.log
for lib in paper_2203_10213_b200/libvkt_b200.so build/y2c5/libvkt_b200.so build/y2c4/libvkt_b200.so; do
  for c in "u8 3 gauss clamp 1024" "u16 3 gauss clamp 1024" "u8 3 gauss clamp 256" "u8 3 gauss wrap 1024"; do
    set -- $c
    VKT_LIB=$PWD/$lib python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --n $5 --reps 9 2>&1 | sed "s|^|[$lib] |"
  done
done > gpurun_out/exp17.log 2>&1
