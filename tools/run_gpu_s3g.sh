# fused level-0 block: epilogue / MMA-warp barrier wait modes (suspend hint, try_wait, test_wait spin)
set -x
mkdir -p gpurun_out/s3g
for rep in 1 2; do for n in base w1 w2 w2m m nomma_w2; do for m in 0 1; do
  echo "== $n vjp$m rep$rep"; timeout 120 ./tools/rbf_prof_$n $m > gpurun_out/s3g/rbf_${n}_vjp${m}_r$rep.txt 2>&1; sed -n 3p gpurun_out/s3g/rbf_${n}_vjp${m}_r$rep.txt; tail -1 gpurun_out/s3g/rbf_${n}_vjp${m}_r$rep.txt
done; done; done
