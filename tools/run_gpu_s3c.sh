# fused level-0 block: wrapped windows as one N = 128 MMA (sw0, kept design) vs two MMAs (sw1)
set -x
mkdir -p gpurun_out/s3c
for rep in 1 2; do for v in 0 1; do for m in 0 1; do
  echo "== sw$v vjp$m rep$rep"; timeout 120 ./tools/rbf_prof_sw$v $m > gpurun_out/s3c/rbf_sw${v}_vjp${m}_r$rep.txt 2>&1; head -3 gpurun_out/s3c/rbf_sw${v}_vjp${m}_r$rep.txt; tail -1 gpurun_out/s3c/rbf_sw${v}_vjp${m}_r$rep.txt
done; done; done
