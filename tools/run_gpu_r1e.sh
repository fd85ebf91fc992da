set -x
timeout 300 python tools/one_iter.py > gpurun_out/one_iter_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 1 -c 2 -o gpurun_out/prof_l0 python tools/one_iter.py > gpurun_out/ncu_l0.log 2>&1; echo $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 11 -c 1 -o gpurun_out/prof_l2 python tools/one_iter.py > gpurun_out/ncu_l2.log 2>&1; echo $?
timeout 900 ncu --set full --clock-control none -k regex:conv_tc -s 0 -c 72 -o /tmp/prof_all python tools/one_iter.py > gpurun_out/ncu_all.log 2>&1; echo $?
ncu -i /tmp/prof_all.ncu-rep --page raw --csv > gpurun_out/prof_all_raw.csv 2>/dev/null
ls -la gpurun_out
