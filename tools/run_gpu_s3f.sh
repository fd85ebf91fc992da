# fused level-0 block bisection: MMAs off / epilogue work off / both (timing only)
set -x
mkdir -p gpurun_out/s3f
for rep in 1 2; do for n in base nomma noepi skel; do for m in 0 1; do
  echo "== $n vjp$m rep$rep"; timeout 120 ./tools/rbf_prof_$n $m > gpurun_out/s3f/rbf_${n}_vjp${m}_r$rep.txt 2>&1; sed -n 3p gpurun_out/s3f/rbf_${n}_vjp${m}_r$rep.txt; tail -1 gpurun_out/s3f/rbf_${n}_vjp${m}_r$rep.txt
done; done; done
