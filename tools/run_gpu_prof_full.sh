# ncu --set full of every network launch (+ the update kernel) of one eager C3 iteration
mkdir -p gpurun_out
timeout 300 python tools/one_iter.py > gpurun_out/one_iter_plain.log 2>&1 && \
timeout 1500 ncu -f --set full --import-source on --clock-control none -k regex:"conv_tc|img2feat|pointwise" -s 0 -c 73 \
  -o /tmp/prof_all python tools/one_iter.py > gpurun_out/ncu_all.log 2>&1; echo full $?
ncu -i /tmp/prof_all.ncu-rep --page raw --csv > gpurun_out/prof_all_raw.csv 2>/dev/null; wc -l gpurun_out/prof_all_raw.csv
