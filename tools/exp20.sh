export VKT_PARITY_LOG=gpurun_out/parity_r02d.jsonl
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/gputest_d.log 2>&1
echo rc=$? >> gpurun_out/gputest_d.log
for c in "u8 3 gauss clamp 1024" "u16 3 gauss clamp 1024" "u8 3 gauss wrap 1024" "u16 3 gauss mirror 512" "u8 3 gauss border 512" "u8 3 gauss clamp 256"; do
  set -- $c
  python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --n $5 --reps 9 2>&1
done > gpurun_out/exp20.log 2>&1
bash tools/ncu_cases.sh r02h "u8 3 gauss clamp 1024" "u16 3 gauss clamp 1024"
bash tools/checked_suite.sh
