set -x
timeout 300 python tools/one_iter.py > gpurun_out/one_iter_plain.log 2>&1 && timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:conv_tc -s 0 -c 1 -o gpurun_out/prof_row python tools/one_iter.py > gpurun_out/ncu_row.log 2>&1; echo $?
