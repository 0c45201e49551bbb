# cfg4 re-measure + ncu, CPU baseline sweep, bench spawn path (gloo, 2 ranks on one GPU)
python tools/profile_case.py --fmt f32 --k 3 --kernel lap --mode wrap --n 2048 --reps 7 > gpurun_out/cfg4.log 2>&1
python tools/baseline_configs.py > gpurun_out/baseline_configs.jsonl 2> gpurun_out/baseline_configs.err
bash tools/ncu_cases.sh r02f "f32 3 lap wrap 2048" "u16 7 gauss clamp 1024" "u8 3 gauss clamp 1024" "f32 3 gauss clamp 1024" "f32 7 gauss clamp 1024"
python tools/cpu_baseline_sweep.py > gpurun_out/cpu_baseline_sweep.txt 2>&1
timeout 600 python bench.py --gpus 2 --test-single-gpu --steps 3 --warmup 3 --no-extra --no-cpu --no-e2e > gpurun_out/bench_spawn2.log 2> gpurun_out/bench_spawn2.err
echo rc=$? >> gpurun_out/bench_spawn2.log
