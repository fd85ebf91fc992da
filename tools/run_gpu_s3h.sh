# fused level-0 block: the saved activation stored by TMA from the u ring (forward)
set -x
mkdir -p gpurun_out/s3h
for rep in 1 2; do for n in base tma tma_nomma; do for m in 0; do
  echo "== $n vjp$m rep$rep"; timeout 120 ./tools/rbf_prof_$n $m > gpurun_out/s3h/rbf_${n}_vjp${m}_r$rep.txt 2>&1; sed -n 3p gpurun_out/s3h/rbf_${n}_vjp${m}_r$rep.txt; tail -1 gpurun_out/s3h/rbf_${n}_vjp${m}_r$rep.txt
done; done; done
timeout 600 python -m pytest tests/test_gpu_rbf.py -q -x -p no:cacheprovider > gpurun_out/s3h/rbf_tests.log 2>&1; tail -2 gpurun_out/s3h/rbf_tests.log
timeout 400 python bench.py --steps 30 --no-cpu-baseline --no-tol-run > gpurun_out/s3h/bench_C3.log 2>&1; tail -1 gpurun_out/s3h/bench_C3.log | cut -c1-250
