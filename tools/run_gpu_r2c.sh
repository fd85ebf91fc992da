set -x
timeout 60 ./tools/tmem_a_probe > gpurun_out/tmem_a_probe.log 2>&1; cat gpurun_out/tmem_a_probe.log
timeout 1200 python -m pytest tests/test_gpu_rician.py tests/test_gpu_livelist.py tests/test_gpu_plan.py tests/test_gpu_layers.py -k "not bf16-simt" -q -p no:cacheprovider > gpurun_out/gpu_tests_r2c.log 2>&1; tail -15 gpurun_out/gpu_tests_r2c.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2c.log 2>&1; tail -1 gpurun_out/bench_r2c.log | cut -c1-2500
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --precision fp32 --no-tol-run > gpurun_out/bench_r2c_fp32.log 2>&1; tail -1 gpurun_out/bench_r2c_fp32.log | cut -c1-2500
