timeout 200 python tools/rbf_dbg.py 2>&1 | grep -c "bad 0"
timeout 150 python -m pytest tests/test_gpu_rbf.py -q -p no:cacheprovider 2>&1 | grep -E "Error|assert|passed|failed" | head -6
FUSE=1 ITERS=1 python tools/one_iter.py >/dev/null 2>&1 && FUSE=1 ITERS=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rbf_launch.csv python tools/one_iter.py > /dev/null 2>&1; echo done
