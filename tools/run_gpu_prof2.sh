set -x
timeout 300 python tools/one_iter.py > gpurun_out/one_iter_plain.log 2>&1 && timeout 900 ncu -f --set full --clock-control none -k regex:"conv_tc|img2feat" -s 0 -c 72 -o /tmp/prof_all python tools/one_iter.py > gpurun_out/ncu_all.log 2>&1; echo full $?
ncu -i /tmp/prof_all.ncu-rep --page raw --csv > gpurun_out/prof_all_raw.csv 2>/dev/null
