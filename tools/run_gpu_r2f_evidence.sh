# Round-2 final evidence (r2f tree): GPU suite, smoke, bench lines for every config, oracle arm, ncu launch lists, stage profiles
set -x
mkdir -p gpurun_out/ev7
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/ev7/smi.txt
timeout 400 python bench.py > gpurun_out/ev7/bench_C3.log 2>&1; tail -1 gpurun_out/ev7/bench_C3.log | cut -c1-300
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/ev7/gpu_tests.log 2>&1; tail -3 gpurun_out/ev7/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev7/smoke.log 2>&1; tail -2 gpurun_out/ev7/smoke.log
timeout 400 python bench.py > gpurun_out/ev7/bench_C3b.log 2>&1; tail -1 gpurun_out/ev7/bench_C3b.log | cut -c1-300
for c in C1 C2 C4; do timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/ev7/bench_$c.log 2>&1; tail -1 gpurun_out/ev7/bench_$c.log | cut -c1-200; done
timeout 400 python bench.py --precision fp32 --steps 10 --no-cpu-baseline > gpurun_out/ev7/bench_C3_fp32.log 2>&1; tail -1 gpurun_out/ev7/bench_C3_fp32.log | cut -c1-200
timeout 600 python bench.py --config C5 --batch 64 --steps 5 --no-cpu-baseline --no-tol-run > gpurun_out/ev7/bench_C5_64.log 2>&1; tail -1 gpurun_out/ev7/bench_C5_64.log | cut -c1-200
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-tol-run > gpurun_out/ev7/bench_C5_512.log 2>&1; tail -1 gpurun_out/ev7/bench_C5_512.log | cut -c1-200
timeout 400 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/ev7/bench_ref.log 2>&1; tail -1 gpurun_out/ev7/bench_ref.log | cut -c1-200
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-tol-run > gpurun_out/ev7/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/ev7/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-tol-run > gpurun_out/ev7/ncu_bench.log 2>&1; echo list $?
timeout 300 python tools/one_iter.py > gpurun_out/ev7/one_iter_C3.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ev7/launches_C3.csv python tools/one_iter.py > gpurun_out/ev7/ncu_C3.log 2>&1; echo ncu C3 $?
for c in C2 C4; do CFG=$c timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ev7/launches_$c.csv python tools/one_iter.py > gpurun_out/ev7/ncu_$c.log 2>&1; echo ncu $c $?; done
CFG=C5 BATCH=64 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ev7/launches_C5.csv python tools/one_iter.py > gpurun_out/ev7/ncu_C5.log 2>&1; echo ncu C5 $?
timeout 120 tools/tiny_prof > gpurun_out/ev7/tiny_prof.txt 2>&1; head -3 gpurun_out/ev7/tiny_prof.txt
for d in 0 1; do timeout 60 tools/rbf_prof $d > gpurun_out/ev7/rbf_prof_$d.txt 2>&1; tail -1 gpurun_out/ev7/rbf_prof_$d.txt; done
