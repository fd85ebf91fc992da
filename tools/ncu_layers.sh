python tools/one_iter.py > gpurun_out/one_iter_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 0 -c 2 -o gpurun_out/prof_l0 python tools/one_iter.py > gpurun_out/ncu_l0.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 10 -c 2 -o gpurun_out/prof_l2 python tools/one_iter.py > gpurun_out/ncu_l2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 15 -c 2 -o gpurun_out/prof_l3 python tools/one_iter.py > gpurun_out/ncu_l3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"img2feat|feat2img" -s 0 -c 2 -o gpurun_out/prof_ht python tools/one_iter.py > gpurun_out/ncu_ht.log 2>&1
ls -la gpurun_out/*.ncu-rep
