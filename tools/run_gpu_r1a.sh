# Round-1 re-entry: full GPU test suite, smoke, bench, ncu launch list + full captures.
# ncu reports are reduced to CSV on the box (gpurun copies back at most 64 MiB).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/gpu_tests.log 2>&1; tail -15 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py --steps 30 --warmup 3 > gpurun_out/bench.log 2>&1; tail -2 gpurun_out/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1; echo ncu_list $?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"conv_tc" -s 0 -c 72 -o /tmp/prof_tc python tools/one_iter.py > gpurun_out/ncu_full.log 2>&1; echo ncu_full $?
ncu -i /tmp/prof_tc.ncu-rep --page raw --csv > gpurun_out/prof_tc_raw.csv 2>/dev/null; echo raw $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"conv_tc" -s 1 -c 1 -o gpurun_out/prof_tc_one python tools/one_iter.py > gpurun_out/ncu_one.log 2>&1; echo ncu_one $?
timeout 600 ncu --set full --clock-control none -k regex:"im2col|step|finalize|advance" -s 0 -c 8 -o /tmp/prof_misc python tools/one_iter.py > gpurun_out/ncu_misc.log 2>&1; echo ncu_misc $?
ncu -i /tmp/prof_misc.ncu-rep --page raw --csv > gpurun_out/prof_misc_raw.csv 2>/dev/null
ls -la gpurun_out/; du -sh gpurun_out
