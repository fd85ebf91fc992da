# fused level-0 block: TMEM blocks handed back right after the drain (early free)
set -x
mkdir -p gpurun_out/s3i
for rep in 1 2; do for n in tma ef ef_nomma ef_noepi; do for m in 0 1; do
  echo "== $n vjp$m rep$rep"; timeout 120 ./tools/rbf_prof_$n $m > gpurun_out/s3i/rbf_${n}_vjp${m}_r$rep.txt 2>&1; sed -n 3p gpurun_out/s3i/rbf_${n}_vjp${m}_r$rep.txt; tail -1 gpurun_out/s3i/rbf_${n}_vjp${m}_r$rep.txt
done; done; done
timeout 600 python -m pytest tests/test_gpu_rbf.py -q -x -p no:cacheprovider > gpurun_out/s3i/rbf_tests.log 2>&1; tail -2 gpurun_out/s3i/rbf_tests.log
timeout 400 python bench.py --steps 30 --no-cpu-baseline --no-tol-run > gpurun_out/s3i/bench_C3.log 2>&1; tail -1 gpurun_out/s3i/bench_C3.log | cut -c1-250
