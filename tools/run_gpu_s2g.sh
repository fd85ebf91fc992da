set -x
mkdir -p gpurun_out/s2g
timeout 600 python -m pytest tests/test_gpu_rbf.py -q -x -p no:cacheprovider > gpurun_out/s2g/rbf_tests.log 2>&1; tail -3 gpurun_out/s2g/rbf_tests.log
timeout 60 tools/rbf_prof 0 > gpurun_out/s2g/rbf_prof_fwd.txt 2>&1; cat gpurun_out/s2g/rbf_prof_fwd.txt
timeout 60 tools/rbf_prof 1 > gpurun_out/s2g/rbf_prof_vjp.txt 2>&1; head -3 gpurun_out/s2g/rbf_prof_vjp.txt; tail -1 gpurun_out/s2g/rbf_prof_vjp.txt
ITERS=50 timeout 300 python tools/rbf_ab.py > gpurun_out/s2g/rbf_ab.txt 2>&1; cat gpurun_out/s2g/rbf_ab.txt
timeout 400 python bench.py --steps 30 --no-cpu-baseline --no-tol-run > gpurun_out/s2g/bench_C3.log 2>&1; tail -1 gpurun_out/s2g/bench_C3.log | cut -c1-250
