set -x
timeout 240 python -m pytest tests/test_gpu_layers.py -q -p no:cacheprovider -x -k "bf16-tc and 0-64-128" > gpurun_out/gpu_layers.log 2>&1; tail -15 gpurun_out/gpu_layers.log
