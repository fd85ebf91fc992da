# round-1 final evidence: full GPU suite, smoke, bench (cpu baseline + tolerance run), reference arm,
# launch list of the bench command, ncu --set full of every network launch of one iteration
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --steps 30 --warmup 3 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-150
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-150
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-tol-run > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-tol-run > gpurun_out/ncu_list.log 2>&1; echo list $?
timeout 300 python tools/one_iter.py > gpurun_out/one_iter_plain.log 2>&1 && timeout 1200 ncu -f --set full --clock-control none -k regex:"conv_tc|img2feat|pointwise" -s 0 -c 73 -o /tmp/prof_all6 python tools/one_iter.py > gpurun_out/ncu_all.log 2>&1; echo full $?
ncu -i /tmp/prof_all6.ncu-rep --page raw --csv > gpurun_out/prof_all_raw.csv 2>/dev/null; wc -l gpurun_out/prof_all_raw.csv
