# ncu --set full of every tcgen05 conv / fused-block launch of one eager C3 iteration (roofline.traffic), C3 fp32 line
mkdir -p gpurun_out/s4f
timeout 400 python bench.py --precision fp32 --steps 10 --no-cpu-baseline > gpurun_out/s4f/bench_C3_fp32.log 2>&1; tail -1 gpurun_out/s4f/bench_C3_fp32.log | cut -c1-200
timeout 1500 ncu -f --set full --clock-control none -k regex:"conv_tc|rbf_kernel" -c 80 \
  -o /tmp/prof_all python tools/one_iter.py > gpurun_out/s4f/ncu_all.log 2>&1; echo full $?
ncu -i /tmp/prof_all.ncu-rep --page raw --csv > gpurun_out/s4f/net_raw.csv 2>/dev/null; wc -l gpurun_out/s4f/net_raw.csv
