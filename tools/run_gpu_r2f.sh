set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -k "tiny or C1" -q -p no:cacheprovider -x > gpurun_out/gpu_tests_r2f.log 2>&1; tail -15 gpurun_out/gpu_tests_r2f.log
timeout 300 python bench.py --config C1 --steps 100 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2f_C1.log 2>&1; tail -1 gpurun_out/bench_r2f_C1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], json.dumps(d['roofline']), d.get('ms_to_tolerance'))"
