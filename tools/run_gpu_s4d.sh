mkdir -p gpurun_out/s4d
timeout 900 python -m pytest tests/test_gpu_layers.py tests/test_gpu_livelist.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/s4d/tests.log 2>&1; tail -2 gpurun_out/s4d/tests.log
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-tol-run > gpurun_out/s4d/bench_C3_$i.log 2>&1; tail -1 gpurun_out/s4d/bench_C3_$i.log | cut -c1-200; done
timeout 600 python bench.py --config C5 --batch 64 --steps 5 --no-cpu-baseline --no-tol-run > gpurun_out/s4d/bench_C5_64.log 2>&1; tail -1 gpurun_out/s4d/bench_C5_64.log | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s4d/launches_C3.csv python tools/one_iter.py > gpurun_out/s4d/ncu_C3.log 2>&1; echo ncu C3 $?
CFG=C5 BATCH=64 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"img2feat|rblur" --clock-control none --csv --log-file gpurun_out/s4d/launches_C5.csv python tools/one_iter.py > gpurun_out/s4d/ncu_C5.log 2>&1; echo ncu C5 $?
grep img2feat gpurun_out/s4d/launches_C3.csv gpurun_out/s4d/launches_C5.csv | grep duration | awk -F'","' '{print $8, $NF}'
