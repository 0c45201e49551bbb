python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edges.py tests/test_gpu_shard.py -q -p no:cacheprovider > gpurun_out/exp3_tests.log 2>&1
echo rc=$? >> gpurun_out/exp3_tests.log
bash tools/ncu_cases.sh r02b "u8 3 gauss clamp 1024"
