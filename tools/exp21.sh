VKT_LIB=$PWD/build/big/libvkt_b200.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edges.py -q -p no:cacheprovider -x 2>&1 | tail -2 > gpurun_out/exp21_tests.log
for lib in paper_2203_10213_b200/libvkt_b200.so build/big/libvkt_b200.so; do
  for c in "u8 3 gauss clamp 1024" "u16 3 gauss clamp 1024" "u8 3 gauss wrap 1024" "u8 3 gauss clamp 256"; do
    set -- $c
    VKT_LIB=$PWD/$lib timeout 120 python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --n $5 --reps 9 2>&1 | sed "s|^|[$lib] |"
  done
done > gpurun_out/exp21.log 2>&1
