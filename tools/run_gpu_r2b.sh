# round 2: 3xTF32 tensor-core path + planner + class timing
set -x
timeout 600 python -m pytest tests/test_gpu_layers.py -q -p no:cacheprovider -k "fp32-tc" -x > gpurun_out/x3_layers.log 2>&1; tail -25 gpurun_out/x3_layers.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/gpu_tests_r2b.log 2>&1; tail -40 gpurun_out/gpu_tests_r2b.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2b.log 2>&1; tail -3 gpurun_out/bench_r2b.log | cut -c1-3000
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --precision fp32 > gpurun_out/bench_r2b_fp32.log 2>&1; tail -3 gpurun_out/bench_r2b_fp32.log | cut -c1-3000
