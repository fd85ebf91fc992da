# round 2, first check: full GPU suite (no -x: see every failure), C3 per-image stops, bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python tools/c3_stop_iters.py > gpurun_out/c3_stop_iters.json 2> gpurun_out/c3_stop_iters.err; tail -c 600 gpurun_out/c3_stop_iters.json
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > gpurun_out/gpu_tests_r2a.log 2>&1; tail -40 gpurun_out/gpu_tests_r2a.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2a.log 2>&1; tail -1 gpurun_out/bench_r2a.log | cut -c1-400
