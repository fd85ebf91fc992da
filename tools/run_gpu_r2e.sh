set -x
timeout 300 python tools/x3_accuracy.py > gpurun_out/x3_accuracy2.log 2>&1; cat gpurun_out/x3_accuracy2.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rician.py -k "tiny or fp32 or rician" -q -p no:cacheprovider -x > gpurun_out/gpu_tests_r2e.log 2>&1; tail -15 gpurun_out/gpu_tests_r2e.log
timeout 300 python bench.py --config C1 --steps 100 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2e_C1.log 2>&1; tail -1 gpurun_out/bench_r2e_C1.log | cut -c1-1500
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --precision fp32 --no-tol-run > gpurun_out/bench_r2e_fp32.log 2>&1; tail -1 gpurun_out/bench_r2e_fp32.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], json.dumps(d['roofline'])[:800])"
