# FFT passes: full-period twiddle table, constant W_32, 3 column blocks per SM
set -x
mkdir -p gpurun_out/s3b
timeout 300 ./tools/tiny_prof > gpurun_out/s3b/tiny_prof.txt 2>&1; head -14 gpurun_out/s3b/tiny_prof.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mri.py -q -x -p no:cacheprovider -k "fft or fidelity or C4 or C5 or mri or phase" > gpurun_out/s3b/fft_tests.log 2>&1; tail -2 gpurun_out/s3b/fft_tests.log
CFG=C5 BATCH=64 timeout 300 python tools/one_iter.py > gpurun_out/s3b/one_C5.log 2>&1; tail -1 gpurun_out/s3b/one_C5.log | cut -c1-200
CFG=C5 BATCH=64 timeout 900 ncu -k regex:"rblur|rphase" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s3b/launches_C5_fft.csv python tools/one_iter.py > gpurun_out/s3b/ncu_C5.log 2>&1; echo ncu C5 $?
CFG=C4 timeout 900 ncu -k regex:"rblur|rphase" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s3b/launches_C4_fft.csv python tools/one_iter.py > gpurun_out/s3b/ncu_C4.log 2>&1; echo ncu C4 $?
timeout 400 python bench.py --config C4 --steps 20 --no-cpu-baseline --no-tol-run > gpurun_out/s3b/bench_C4.log 2>&1; tail -1 gpurun_out/s3b/bench_C4.log | cut -c1-200
