# fused level-0 VJP block: bulk L2 prefetch of the saved activation rows
set -x
mkdir -p gpurun_out/s3j
for rep in 1 2; do for n in tma pf pf_nomma; do for m in 1 0; do
  echo "== $n vjp$m rep$rep"; timeout 120 ./tools/rbf_prof_$n $m > gpurun_out/s3j/rbf_${n}_vjp${m}_r$rep.txt 2>&1; sed -n 3p gpurun_out/s3j/rbf_${n}_vjp${m}_r$rep.txt
done; done; done
timeout 600 python -m pytest tests/test_gpu_rbf.py -q -x -p no:cacheprovider > gpurun_out/s3j/rbf_tests.log 2>&1; tail -2 gpurun_out/s3j/rbf_tests.log
timeout 400 python bench.py --steps 30 --no-cpu-baseline --no-tol-run > gpurun_out/s3j/bench_C3.log 2>&1; tail -1 gpurun_out/s3j/bench_C3.log | cut -c1-250
timeout 300 python tools/one_iter.py > gpurun_out/s3j/one.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s3j/launches_C3.csv python tools/one_iter.py > gpurun_out/s3j/ncu_C3.log 2>&1; echo ncu $?
