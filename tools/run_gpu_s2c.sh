set -x
mkdir -p gpurun_out/s2c
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "tiny or C1" > gpurun_out/s2c/tiny_tests.log 2>&1; tail -5 gpurun_out/s2c/tiny_tests.log
timeout 120 tools/tiny_prof > gpurun_out/s2c/tiny_prof.txt 2>&1; cat gpurun_out/s2c/tiny_prof.txt
timeout 400 python bench.py --config C1 --no-cpu-baseline > gpurun_out/s2c/bench_C1.log 2>&1; tail -1 gpurun_out/s2c/bench_C1.log | cut -c1-300
