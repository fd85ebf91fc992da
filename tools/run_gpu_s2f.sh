set -x
mkdir -p gpurun_out/s2f
timeout 900 python -m pytest tests/test_gpu_layers.py -q -x -p no:cacheprovider > gpurun_out/s2f/layers.log 2>&1; tail -3 gpurun_out/s2f/layers.log
timeout 400 python bench.py --steps 30 --no-cpu-baseline --no-tol-run > gpurun_out/s2f/bench_C3.log 2>&1; tail -1 gpurun_out/s2f/bench_C3.log | cut -c1-250
timeout 300 python tools/one_iter.py > gpurun_out/s2f/one_iter.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s2f/launches_C3.csv python tools/one_iter.py > gpurun_out/s2f/ncu.log 2>&1; echo ncu $?
