export VKT_LIB=$PWD/build/sep2/libvkt_b200.so
for c in "u16 7 border 64" "u16 7 clamp 16" "u16 7 clamp 64" "u16 7 mirror 64" "u16 5 clamp 64" "u8 3 clamp 64" "f32 7 clamp 64" "u16 7 wrap 64"; do
  set -- $c
  timeout 30 python tools/dbg_sep2.py $1 $2 $3 $4 > /tmp/o.txt 2>&1; echo "rc=$? $c $(tail -1 /tmp/o.txt)"
done
timeout 300 python -m pytest tests/test_gpu_separable.py -x -q -p no:cacheprovider 2>&1 | tail -3
unset VKT_LIB
for lib in "" build/sep2/libvkt_b200.so; do
  for c in "u8 3 gauss clamp" "u16 3 gauss clamp" "u16 5 gauss clamp" "u16 7 gauss clamp" "u16 7 gauss border" "f32 7 gauss clamp" "u16 9 gauss clamp" "f32 5 box clamp"; do
    set -- $c
    VKT_LIB=${lib:+$PWD/$lib} timeout 60 python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --n 1024 --reps 7 2>&1 | tail -1 | sed "s|^|[$lib] |; s/dims=(1024, 1024, 1024)//; s/(all.*//"
  done
done
