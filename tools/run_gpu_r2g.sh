set -x
./tools/tiny_prof 2>&1 | tail -14
timeout 600 python -m pytest tests/test_gpu_parity.py -k "tiny or C1" -q -p no:cacheprovider -x > gpurun_out/gpu_tests_r2g.log 2>&1; tail -5 gpurun_out/gpu_tests_r2g.log
