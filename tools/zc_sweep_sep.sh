# z-chunk depth sweep of the separable kernel (VKT_TMA_ZC overrides the model)
for c in "u16 7 gauss" "u8 3 gauss" "f32 5 box" "u16 9 gauss"; do
  set -- $c
  for zc in 0 64 96 128 171 205 256 342 512; do
    if [ $zc = 0 ]; then unset VKT_TMA_ZC; else export VKT_TMA_ZC=$zc; fi
    timeout 60 python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode clamp --n 1024 --reps 9 2>&1 | tail -1 | sed "s|^|[zc=$zc] |; s/(all.*//; s/dims=(1024, 1024, 1024)//"
  done
done
