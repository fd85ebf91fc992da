# round-1 final evidence, call 1 of 3 (no profiler): full GPU suite, smoke, C3 bench (cpu baseline +
# tolerance run), reference arm, C2 / C4 / C5 bench lines, JFB timing
# call 2: tools/run_gpu_prof_list.sh (ncu launch list of the bench command)
# call 3: tools/run_gpu_prof_full.sh (ncu --set full of every network launch of one iteration)
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --steps 30 --warmup 3 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-200
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-200
for c in C2 C4 C5; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; tail -1 gpurun_out/bench_$c.log | cut -c1-160; done
timeout 600 python tools/jfb_bench.py --batch 16 --steps 5 --no-oracle > gpurun_out/jfb.log 2>&1; tail -1 gpurun_out/jfb.log | cut -c1-200
