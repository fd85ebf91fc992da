timeout 900 python -m pytest tests/test_gpu_layers.py -q -x -p no:cacheprovider --timeout 120 > gpurun_out/layers.log 2>&1; tail -2 gpurun_out/layers.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider --timeout 300 > gpurun_out/parity.log 2>&1; tail -2 gpurun_out/parity.log
python tools/one_iter.py > gpurun_out/one_iter_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_it.csv python tools/one_iter.py > gpurun_out/ncu_list.log 2>&1
