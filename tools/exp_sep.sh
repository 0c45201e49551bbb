# y-first separable variant (diagnostics build)
VKT_LIB=$PWD/build/sepy/libvkt_b200.so timeout 300 python -m pytest tests/test_gpu_separable.py -x -q -p no:cacheprovider 2>&1 | tail -3
for lib in "" build/sepy/libvkt_b200.so; do
  for c in "u8 3 gauss clamp" "u16 5 gauss clamp" "u16 7 gauss clamp" "u16 7 gauss border" "f32 7 gauss clamp" "u16 9 gauss clamp" "f32 5 box clamp"; do
    set -- $c
    VKT_LIB=${lib:+$PWD/$lib} timeout 60 python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --n 1024 --reps 7 2>&1 | tail -1 | sed "s|^|[$lib] |; s/dims=(1024, 1024, 1024)//; s/(all.*//"
  done
done
