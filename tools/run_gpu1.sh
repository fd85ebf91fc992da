set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import torch; print(torch.cuda.get_device_name(0))"
timeout 600 python -m pytest tests/test_gpu_layers.py -q -x -k "fp32" -p no:cacheprovider --timeout 120 > gpurun_out/l_fp32.log 2>&1; tail -5 gpurun_out/l_fp32.log
timeout 600 python -m pytest tests/test_gpu_layers.py -q -k "bf16-simt" -p no:cacheprovider --timeout 120 > gpurun_out/l_bsimt.log 2>&1; tail -5 gpurun_out/l_bsimt.log
timeout 300 python -m pytest tests/test_gpu_layers.py -q -x -k "bf16-tc and 0-32-32-20-40-0" -p no:cacheprovider --timeout 60 > gpurun_out/l_tc1.log 2>&1; tail -30 gpurun_out/l_tc1.log
timeout 900 python -m pytest tests/test_gpu_layers.py -q -k "bf16-tc" -p no:cacheprovider --timeout 60 > gpurun_out/l_tc.log 2>&1; tail -30 gpurun_out/l_tc.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 > gpurun_out/parity.log 2>&1; tail -40 gpurun_out/parity.log
