# Final evidence of round 2 (r2g tree: single-wave fused head): whole GPU suite, smoke, default bench twice, C5 / C2 / C4 lines, oracle arm, bench launch list
set -x
mkdir -p gpurun_out/ev8
timeout 400 python bench.py > gpurun_out/ev8/bench_C3.log 2>&1; tail -1 gpurun_out/ev8/bench_C3.log | cut -c1-300
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ev8/gpu_tests.log 2>&1; tail -3 gpurun_out/ev8/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev8/smoke.log 2>&1; tail -2 gpurun_out/ev8/smoke.log
timeout 400 python bench.py > gpurun_out/ev8/bench_C3b.log 2>&1; tail -1 gpurun_out/ev8/bench_C3b.log | cut -c1-300
for c in C1 C2 C4; do timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/ev8/bench_$c.log 2>&1; tail -1 gpurun_out/ev8/bench_$c.log | cut -c1-200; done
timeout 600 python bench.py --config C5 --batch 64 --steps 5 --no-cpu-baseline --no-tol-run > gpurun_out/ev8/bench_C5_64.log 2>&1; tail -1 gpurun_out/ev8/bench_C5_64.log | cut -c1-200
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-tol-run > gpurun_out/ev8/bench_C5_512.log 2>&1; tail -1 gpurun_out/ev8/bench_C5_512.log | cut -c1-200
timeout 400 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/ev8/bench_ref.log 2>&1; tail -1 gpurun_out/ev8/bench_ref.log | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/ev8/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-tol-run > gpurun_out/ev8/ncu_bench.log 2>&1; echo list $?
