# Round-2 evidence: full GPU suite, bench lines for every config, ncu launch lists (time + DRAM bytes)
set -x
mkdir -p gpurun_out/ev
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/ev/smi.txt
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/ev/gpu_tests.log 2>&1; tail -30 gpurun_out/ev/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1; tail -2 gpurun_out/ev/smoke.log
timeout 400 python bench.py > gpurun_out/ev/bench_C3.log 2>&1; tail -1 gpurun_out/ev/bench_C3.log | cut -c1-300
timeout 400 python bench.py --precision fp32 --steps 10 --no-cpu-baseline > gpurun_out/ev/bench_C3_fp32.log 2>&1; tail -1 gpurun_out/ev/bench_C3_fp32.log | cut -c1-200
for c in C1 C2 C4; do timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/ev/bench_$c.log 2>&1; tail -1 gpurun_out/ev/bench_$c.log | cut -c1-200; done
timeout 600 python bench.py --config C5 --batch 64 --steps 5 --no-cpu-baseline --no-tol-run > gpurun_out/ev/bench_C5_64.log 2>&1; tail -1 gpurun_out/ev/bench_C5_64.log | cut -c1-200
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-tol-run > gpurun_out/ev/bench_C5_512.log 2>&1; tail -1 gpurun_out/ev/bench_C5_512.log | cut -c1-200
timeout 400 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/ev/bench_ref.log 2>&1; tail -1 gpurun_out/ev/bench_ref.log | cut -c1-200
for c in C2 C4; do CFG=$c timeout 300 python tools/one_iter.py > gpurun_out/ev/one_iter_$c.log 2>&1 && CFG=$c timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ev/launches_$c.csv python tools/one_iter.py > gpurun_out/ev/ncu_$c.log 2>&1; echo ncu $c $?; done
CFG=C5 BATCH=8 timeout 300 python tools/one_iter.py > gpurun_out/ev/one_iter_C5.log 2>&1 && CFG=C5 BATCH=8 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/ev/launches_C5.csv python tools/one_iter.py > gpurun_out/ev/ncu_C5.log 2>&1; echo ncu C5 $?
