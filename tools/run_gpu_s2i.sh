set -x
mkdir -p gpurun_out/s2i
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mri.py -q -x -p no:cacheprovider -k "fft or C4 or C5 or mri or fidelity" > gpurun_out/s2i/fft_tests.log 2>&1; tail -3 gpurun_out/s2i/fft_tests.log
for c in C4; do CFG=$c timeout 300 python tools/one_iter.py > gpurun_out/s2i/one_$c.log 2>&1; CFG=$c timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s2i/launches_$c.csv python tools/one_iter.py > gpurun_out/s2i/ncu_$c.log 2>&1; echo ncu $c $?; done
CFG=C5 BATCH=64 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:rblur --csv --log-file gpurun_out/s2i/launches_C5.csv python tools/one_iter.py > gpurun_out/s2i/ncu_C5.log 2>&1; echo ncu C5 $?
