set -x
mkdir -p gpurun_out/s2e
timeout 300 python tools/one_iter.py > gpurun_out/s2e/plain.log 2>&1; tail -1 gpurun_out/s2e/plain.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_tc_kernel --launch-skip 4 --launch-count 1 -o gpurun_out/s2e/l1 python tools/one_iter.py > gpurun_out/s2e/ncu_l1.log 2>&1; tail -2 gpurun_out/s2e/ncu_l1.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_tc_kernel --launch-skip 9 --launch-count 1 -o gpurun_out/s2e/l2 python tools/one_iter.py > gpurun_out/s2e/ncu_l2.log 2>&1; tail -2 gpurun_out/s2e/ncu_l2.log
