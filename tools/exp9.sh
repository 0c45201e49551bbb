for zc in 0 2 4 6 8 12; do
  if [ $zc = 0 ]; then unset VKT_TMA_ZC; else export VKT_TMA_ZC=$zc; fi
  python tools/profile_case.py --fmt u8 --k 3 --kernel gauss --mode clamp --n 256 --reps 9 2>&1 | sed "s|^|[zc=$zc] |"
  python tools/profile_case.py --fmt u16 --k 3 --kernel gauss --mode clamp --n 512 --reps 9 2>&1 | sed "s|^|[zc=$zc] |"
done > gpurun_out/exp9.log 2>&1
