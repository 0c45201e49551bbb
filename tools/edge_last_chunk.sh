for c in "u16 7 gauss clamp" "u8 3 gauss clamp" "u16 3 gauss clamp" "f32 7 gauss clamp" "u8 5 gauss clamp"; do
  set -- $c
  timeout 60 python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --n 1024 --reps 9 2>&1 | tail -1 | sed "s/(all.*//; s/dims=(1024, 1024, 1024)//"
done
timeout 120 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:filter_sep -c 1 --csv python tools/profile_case.py --fmt u16 --k 7 --kernel gauss --mode clamp --n 1024 --reps 1 2>/dev/null | grep -E "dram__bytes|hit_rate" | awk -F'","' '{print $(NF-2) " " $(NF-1) " " $NF}'
