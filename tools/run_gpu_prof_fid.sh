# per-launch time + DRAM bytes of the fidelity / update kernels of one eager iteration of C2, C3, C4,
# C5 (one metrics-only ncu kind), after the same command exited 0 without the profiler
mkdir -p gpurun_out
for c in C2 C3 C4 C5; do
  CFG=$c timeout 600 python tools/one_iter.py > gpurun_out/oi_$c.log 2>&1 && \
  CFG=$c timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"blur|phase|pointwise|mri|inpaint" --csv --log-file gpurun_out/fid_$c.csv python tools/one_iter.py \
    > gpurun_out/ncu_fid_$c.log 2>&1; echo $c $?
done
