# ncu --set full with source of the C1 whole-solve kernel (stall reasons per stage)
set -x
mkdir -p gpurun_out/s3e
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tiny_solve -c 1 -o gpurun_out/s3e/tiny python bench.py --config C1 --steps 2 --warmup 3 --no-cpu-baseline --no-tol-run > gpurun_out/s3e/ncu_tiny.log 2>&1; echo ncu tiny $?
