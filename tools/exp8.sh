export VKT_PARITY_LOG=gpurun_out/parity_r02b.jsonl
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/gputest_b.log 2>&1
echo rc=$? >> gpurun_out/gputest_b.log
for c in "u8 3 gauss clamp 1024" "u16 3 gauss clamp 1024" "u8 5 gauss clamp 1024" "u16 5 box clamp 1024" "u16 7 gauss clamp 1024" "u8 3 gauss clamp 256" "u8 5 gauss clamp 512" "u8 5 gauss wrap 512"; do
  set -- $c
  python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --n $5 --reps 7 2>&1
done > gpurun_out/exp8.log 2>&1
