set -x
timeout 300 python -m pytest tests/test_gpu_rbf.py -q -p no:cacheprovider -x > gpurun_out/rbf_tests.log 2>&1; tail -25 gpurun_out/rbf_tests.log
