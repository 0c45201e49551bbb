# separable-kernel variants (diagnostics builds): 6 producer warps at K = 5 / 9
for lib in "" build/pwx5/libvkt_b200.so build/pwx9/libvkt_b200.so; do
  for c in "u8 5 gauss clamp" "u16 5 gauss clamp" "f32 5 box clamp" "u16 9 gauss clamp" "f32 9 gauss clamp"; do
    set -- $c
    VKT_LIB=${lib:+$PWD/$lib} timeout 60 python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --n 1024 --reps 7 2>&1 | tail -1 | sed "s|^|[$lib] |; s/dims=(1024, 1024, 1024)//; s/(all.*//"
  done
done
