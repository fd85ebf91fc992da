# ncu --set full with source of the C1 whole-solve kernel and one fused level-0 block (stall reasons)
set -x
mkdir -p gpurun_out/s3d
timeout 300 python bench.py --config C1 --steps 5 --warmup 3 --no-cpu-baseline --no-tol-run > gpurun_out/s3d/bench_C1.log 2>&1; echo bench $?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tiny_solve -c 1 -o gpurun_out/s3d/tiny python bench.py --config C1 --steps 2 --warmup 1 --no-cpu-baseline --no-tol-run > gpurun_out/s3d/ncu_tiny.log 2>&1; echo ncu tiny $?
timeout 300 python tools/one_iter.py > gpurun_out/s3d/one.log 2>&1; echo one $?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:rbf_kernel -c 1 -o gpurun_out/s3d/rbf python tools/one_iter.py > gpurun_out/s3d/ncu_rbf.log 2>&1; echo ncu rbf $?
ls -la gpurun_out/s3d
