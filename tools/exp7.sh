for zc in 0 32 48 96 128 171 256; do
  for c in "u8 3 gauss clamp 1024" "u16 3 gauss clamp 1024"; do
    set -- $c
    if [ $zc = 0 ]; then unset VKT_TMA_ZC; else export VKT_TMA_ZC=$zc; fi
    python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --n $5 --reps 7 2>&1 | sed "s|^|[zc=$zc] |"
  done
done > gpurun_out/exp7.log 2>&1
