# z-chunk depth vs time and DRAM traffic, separable cfg3 kernel
for zc in 64 96 128; do
  export VKT_TMA_ZC=$zc
  timeout 60 python tools/profile_case.py --fmt u16 --k 7 --kernel gauss --mode clamp --n 1024 --reps 9 2>&1 | tail -1 | sed "s|^|[zc=$zc] |; s/(all.*//; s/dims=(1024, 1024, 1024)//"
  timeout 120 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:filter_sep -c 1 --csv python tools/profile_case.py --fmt u16 --k 7 --kernel gauss --mode clamp --n 1024 --reps 1 2>/dev/null | grep -E "dram__bytes|hit_rate" | awk -F'","' -v z=$zc '{print "[zc=" z "] " $(NF-2) " " $(NF-1) " " $NF}'
done
