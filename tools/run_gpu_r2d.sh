set -x
timeout 60 ./tools/tmem_a_probe > gpurun_out/tmem_a_probe2.log 2>&1; cat gpurun_out/tmem_a_probe2.log
timeout 300 python tools/x3_accuracy.py > gpurun_out/x3_accuracy.log 2>&1; cat gpurun_out/x3_accuracy.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-tol-run > gpurun_out/bench_r2d.log 2>&1; tail -1 gpurun_out/bench_r2d.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], json.dumps(d['roofline']))"
