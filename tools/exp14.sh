for zc in 0 93 128 146 205 256 342 512; do
  if [ $zc = 0 ]; then unset VKT_TMA_ZC; else export VKT_TMA_ZC=$zc; fi
  for c in "u16 7 gauss clamp 1024" "u16 5 box clamp 1024"; do
    set -- $c
    python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --n $5 --reps 7 2>&1 | sed "s|^|[zc=$zc] |"
  done
done > gpurun_out/exp14.log 2>&1
