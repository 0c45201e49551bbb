# separable-kernel variants (diagnostics builds): 1 CTA/SM, 32-row tiles for one K
for lib in "" build/big7/libvkt_b200.so build/big5/libvkt_b200.so; do
  for c in "u16 7 gauss clamp" "u16 7 gauss border" "f32 7 gauss clamp" "u16 5 gauss clamp" "f32 5 box clamp"; do
    set -- $c
    VKT_LIB=${lib:+$PWD/$lib} timeout 60 python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --n 1024 --reps 7 2>&1 | tail -1 | sed "s|^|[$lib] |; s/dims=(1024, 1024, 1024)//; s/(all.*//"
  done
done
