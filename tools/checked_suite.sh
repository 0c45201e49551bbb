# The GPU test suite against the checked build (bounds checks + sync jitter,
# see csrc/common.cuh): stands in for compute-sanitizer, which the pool lacks.
#   python paper_2203_10213_b200/build.py --variant=checked -DVKT_CHECKS -DVKT_JITTER
#   bash tools/checked_suite.sh  -> gpurun_out/checked_suite.log
export VKT_LIB=$PWD/build/checked/libvkt_b200.so
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 \
  --deselect tests/test_gpu_multiproc.py > gpurun_out/checked_suite.log 2>&1
echo "rc=$?" >> gpurun_out/checked_suite.log
for i in 1 2 3; do python tools/sanitize_cases.py >> gpurun_out/checked_suite.log 2>&1; done
echo "rc_cases=$?" >> gpurun_out/checked_suite.log
