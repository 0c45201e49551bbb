for v in rows y4c4; do
  for c in "u8 3 gauss clamp 1024" "u16 3 gauss clamp 1024" "u8 3 gauss clamp 256" "u8 3 gauss wrap 1024" "u16 3 gauss mirror 512"; do
    set -- $c
    VKT_LIB=build/$v/libvkt_b200.so python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --n $5 --reps 7 2>&1 | sed "s/^/$v /"
  done
done > gpurun_out/exp1.log
VKT_LIB=build/y4c4/libvkt_b200.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edges.py -q -p no:cacheprovider -x > gpurun_out/exp1_tests.log 2>&1
