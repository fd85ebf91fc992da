set -x
timeout 900 python -m pytest tests/test_gpu_layers.py tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 600 -x > gpurun_out/gpu_tests.log 2>&1; tail -5 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
python tools/one_iter.py > gpurun_out/one_iter_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_it.csv python tools/one_iter.py > gpurun_out/ncu_list.log 2>&1; echo ncu $?
