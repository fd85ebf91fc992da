timeout 900 python -m pytest tests/test_gpu_layers.py -q -p no:cacheprovider --timeout 120 > gpurun_out/layers.log 2>&1; tail -3 gpurun_out/layers.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 > gpurun_out/parity.log 2>&1; tail -15 gpurun_out/parity.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.log 2>&1; tail -5 gpurun_out/bench.log
