for lib in paper_2203_10213_b200/libvkt_b200.so build/ws4/libvkt_b200.so build/pw3/libvkt_b200.so; do
  VKT_WS=1 VKT_LIB=$PWD/$lib timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -p no:cacheprovider -x 2>&1 | tail -1 | sed "s|^|[$lib tests] |"
  for c in "u8 3 gauss clamp 1024" "u16 3 gauss clamp 1024" "u8 3 gauss wrap 1024"; do
    set -- $c
    VKT_WS=1 VKT_LIB=$PWD/$lib timeout 120 python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --n $5 --reps 9 2>&1 | sed "s|^|[$lib] |"
  done
done > gpurun_out/exp19.log 2>&1
