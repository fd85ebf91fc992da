set -x
mkdir -p gpurun_out/s2l
timeout 400 python bench.py --steps 30 --no-cpu-baseline --no-tol-run > gpurun_out/s2l/bench_C3.log 2>&1; tail -1 gpurun_out/s2l/bench_C3.log | cut -c1-250
timeout 2700 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s2l/gpu_tests.log 2>&1; tail -3 gpurun_out/s2l/gpu_tests.log
timeout 300 python tools/one_iter.py > gpurun_out/s2l/one_iter.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s2l/launches_C3.csv python tools/one_iter.py > gpurun_out/s2l/ncu.log 2>&1; echo ncu $?
