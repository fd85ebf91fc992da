set -x
mkdir -p gpurun_out/s2n
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_livelist.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > gpurun_out/s2n/tests.log 2>&1; tail -3 gpurun_out/s2n/tests.log
timeout 400 python bench.py --steps 30 --no-cpu-baseline --no-tol-run > gpurun_out/s2n/bench_C3.log 2>&1; tail -1 gpurun_out/s2n/bench_C3.log | cut -c1-250
timeout 300 python tools/one_iter.py > gpurun_out/s2n/one_iter.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s2n/launches_C3.csv python tools/one_iter.py > gpurun_out/s2n/ncu.log 2>&1; echo ncu $?
