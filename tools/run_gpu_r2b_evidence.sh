# Round-2 (session 2) evidence on the current tree: GPU suite, smoke, bench lines, launch lists
set -x
mkdir -p gpurun_out/ev3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/ev3/smi.txt
timeout 400 python bench.py > gpurun_out/ev3/bench_C3.log 2>&1; tail -1 gpurun_out/ev3/bench_C3.log | cut -c1-300
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/ev3/gpu_tests.log 2>&1; tail -3 gpurun_out/ev3/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev3/smoke.log 2>&1; tail -2 gpurun_out/ev3/smoke.log
timeout 400 python bench.py > gpurun_out/ev3/bench_C3b.log 2>&1; tail -1 gpurun_out/ev3/bench_C3b.log | cut -c1-300
for c in C1 C2 C4; do timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/ev3/bench_$c.log 2>&1; tail -1 gpurun_out/ev3/bench_$c.log | cut -c1-200; done
timeout 400 python bench.py --precision fp32 --steps 10 --no-cpu-baseline > gpurun_out/ev3/bench_C3_fp32.log 2>&1; tail -1 gpurun_out/ev3/bench_C3_fp32.log | cut -c1-200
timeout 600 python bench.py --config C5 --batch 64 --steps 5 --no-cpu-baseline --no-tol-run > gpurun_out/ev3/bench_C5_64.log 2>&1; tail -1 gpurun_out/ev3/bench_C5_64.log | cut -c1-200
timeout 300 python tools/one_iter.py > gpurun_out/ev3/one_iter_C3.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ev3/launches_C3.csv python tools/one_iter.py > gpurun_out/ev3/ncu_C3.log 2>&1; echo ncu C3 $?
for c in C4; do CFG=$c timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ev3/launches_$c.csv python tools/one_iter.py > gpurun_out/ev3/ncu_$c.log 2>&1; echo ncu $c $?; done
