mkdir -p gpurun_out/s4c
timeout 60 tools/occ_probe > gpurun_out/s4c/occ_probe.txt 2>&1; cat gpurun_out/s4c/occ_probe.txt
timeout 900 ncu --metrics gpu__time_duration.sum,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,launch__grid_size -k regex:img2feat --clock-control none --csv --log-file gpurun_out/s4c/launches_i2f.csv python tools/one_iter.py > gpurun_out/s4c/ncu_C3.log 2>&1; echo ncu C3 $?
grep -c img2feat gpurun_out/s4c/launches_i2f.csv; grep img2feat gpurun_out/s4c/launches_i2f.csv | awk -F'","' '{print $8, $13, $15}'
