for mode in wrap mirror; do for zc in 64 128 0; do
  if [ $zc = 0 ]; then unset VKT_TMA_ZC; else export VKT_TMA_ZC=$zc; fi
  timeout 60 python tools/profile_case.py --fmt u16 --k 7 --kernel gauss --mode $mode --n 1024 --reps 9 2>&1 | tail -1 | sed "s|^|[zc=$zc] |; s/(all.*//; s/dims=(1024, 1024, 1024)//"
done; done
