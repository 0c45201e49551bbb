# separable-kernel variants (diagnostics builds)
for lib in "" build/pred/libvkt_b200.so; do
  for c in "u8 3 gauss clamp" "u16 7 gauss clamp" "u16 7 gauss border" "f32 7 gauss clamp" "u16 9 gauss clamp"; do
    set -- $c
    VKT_LIB=${lib:+$PWD/$lib} timeout 120 python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --n 1024 --reps 7 2>&1 | tail -1 | sed "s|^|[$lib] |; s/dims=(1024, 1024, 1024)//; s/(all.*//"
  done
done
