python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -p no:cacheprovider > gpurun_out/exp11_tests.log 2>&1
echo rc=$? >> gpurun_out/exp11_tests.log
python tools/aniso_rates.py 512 > gpurun_out/aniso_rates.jsonl 2> gpurun_out/aniso_rates.err
