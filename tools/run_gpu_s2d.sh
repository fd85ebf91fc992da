set -x
mkdir -p gpurun_out/s2d
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tiny_solve -c 1 -o gpurun_out/s2d/tiny python bench.py --config C1 --steps 2 --warmup 3 --no-cpu-baseline --no-tol-run > gpurun_out/s2d/ncu.log 2>&1; tail -3 gpurun_out/s2d/ncu.log
ls -la gpurun_out/s2d
