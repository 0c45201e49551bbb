export VKT_PARITY_LOG=gpurun_out/parity_r02c.jsonl
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/gputest_c.log 2>&1
echo rc=$? >> gpurun_out/gputest_c.log
python tools/baseline_configs.py > gpurun_out/baseline_configs.jsonl 2> gpurun_out/baseline_configs.err
for c in "f32 3 gauss clamp 1024" "f32 3 gauss wrap 1024" "f32 3 gauss border 1024" "f32 3 gauss mirror 1024" "f32 5 box clamp 1024" "f32 7 gauss clamp 1024"; do
  set -- $c
  python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --n $5 --reps 7 2>&1
done > gpurun_out/exp12.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c.log 2>&1
echo rc=$? >> gpurun_out/bench_c.log
