# ncu launch list (per-launch device time, clocks not locked) of the bench command, after the same
# command exited 0 without the profiler
mkdir -p gpurun_out
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-tol-run > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-tol-run > gpurun_out/ncu_list.log 2>&1; echo list $?
