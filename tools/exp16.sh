python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_shard.py -q -p no:cacheprovider > gpurun_out/exp16_tests.log 2>&1
echo rc=$? >> gpurun_out/exp16_tests.log
python tools/aniso_rates.py 512 > gpurun_out/aniso_rates2.jsonl 2> gpurun_out/aniso_rates2.err
