# quick check: tcgen05 layer parity, bf16 parity subset, bench, launch list of one iteration
set -x
timeout 400 python -m pytest tests/test_gpu_layers.py -q -p no:cacheprovider -x -k "bf16-tc" > gpurun_out/gpu_layers.log 2>&1; tail -2 gpurun_out/gpu_layers.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "bf16 or grad_g or determinism" > gpurun_out/gpu_parity.log 2>&1; tail -2 gpurun_out/gpu_parity.log
timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-200
timeout 300 python tools/one_iter.py > gpurun_out/one_iter_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_it.csv python tools/one_iter.py > gpurun_out/ncu_list.log 2>&1; echo ncu $?
