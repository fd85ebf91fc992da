# ncu --set full of the head (img2feat) and the tail / head-adjoint (EPI_IMG) launches of one eager C3 iteration
mkdir -p gpurun_out/s4a
timeout 300 python tools/one_iter.py > gpurun_out/s4a/plain.log 2>&1 && \
timeout 900 ncu -f --set full --import-source on --clock-control none --launch-skip 32 --launch-count 2 \
  -o gpurun_out/s4a/headtail python tools/one_iter.py > gpurun_out/s4a/ncu.log 2>&1; echo full $?
ncu -i gpurun_out/s4a/headtail.ncu-rep --page raw --csv > gpurun_out/s4a/headtail_raw.csv 2>/dev/null
ncu -i gpurun_out/s4a/headtail.ncu-rep --page details > gpurun_out/s4a/headtail_details.txt 2>/dev/null
ncu -i gpurun_out/s4a/headtail.ncu-rep --page source --csv --print-source sass > gpurun_out/s4a/headtail_source.csv 2>/dev/null
wc -l gpurun_out/s4a/*
# the driver's N = 1 launch form under torch.distributed.run (env-var path of bench.py)
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline --no-tol-run > gpurun_out/s4a/bench_torchrun_n1.log 2>&1; tail -1 gpurun_out/s4a/bench_torchrun_n1.log | cut -c1-200
