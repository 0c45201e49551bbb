for mode in wrap clamp; do for zc in 64 128; do
  export VKT_TMA_ZC=$zc
  timeout 60 python tools/profile_case.py --fmt u16 --k 7 --kernel gauss --mode $mode --n 1024 --reps 9 2>&1 | tail -1 | sed "s|^|[zc=$zc] |; s/(all.*//; s/dims=(1024, 1024, 1024)//"
done; done
unset VKT_TMA_ZC
for mode in wrap clamp mirror; do
  timeout 120 python tools/profile_case.py --fmt f32 --k 3 --kernel lap --mode $mode --n 1024 --reps 9 2>&1 | tail -1 | sed "s/(all.*//"
done
timeout 300 python tools/profile_case.py --fmt f32 --k 3 --kernel lap --mode wrap --n 2048 --reps 5 2>&1 | tail -1 | sed "s/(all.*//"
