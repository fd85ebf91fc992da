# C1 kernel with all 512 threads in the 16->16 stages; K = max_iter fp32 trajectories
set -x
mkdir -p gpurun_out/s3a
timeout 300 ./tools/tiny_prof > gpurun_out/s3a/tiny_prof.txt 2>&1; cat gpurun_out/s3a/tiny_prof.txt | head -16
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "tiny_whole or C1" > gpurun_out/s3a/tiny_tests.log 2>&1; tail -2 gpurun_out/s3a/tiny_tests.log
timeout 300 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/s3a/bench_C1.log 2>&1; tail -1 gpurun_out/s3a/bench_C1.log | cut -c1-330
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "max_iter" --durations=10 > gpurun_out/s3a/maxiter.log 2>&1; tail -15 gpurun_out/s3a/maxiter.log
