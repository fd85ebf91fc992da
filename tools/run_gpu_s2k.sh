set -x
mkdir -p gpurun_out/s2k
timeout 1200 python -m pytest tests/test_gpu_jfb.py -q -x -p no:cacheprovider > gpurun_out/s2k/jfb_tests.log 2>&1; tail -3 gpurun_out/s2k/jfb_tests.log
timeout 600 python tools/jfb_bench.py --config C3 --batch 16 --steps 5 --warmup 2 > gpurun_out/s2k/jfb_bench.log 2>&1; tail -2 gpurun_out/s2k/jfb_bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2k/jfb_launches.csv python tools/jfb_bench.py --batch 4 --steps 1 --warmup 0 --no-oracle > gpurun_out/s2k/ncu.log 2>&1; echo ncu $?
