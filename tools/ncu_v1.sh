# launch list (cold-cache serialised device times) + full capture of a few tcgen05 conv launches
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
python tools/one_iter.py > gpurun_out/one_iter_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 0 -c 8 -o gpurun_out/prof_tc python tools/one_iter.py > gpurun_out/ncu_full.log 2>&1
python tools/one_iter.py > gpurun_out/one_iter_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"feat2img|img2feat" -s 0 -c 4 -o gpurun_out/prof_ht python tools/one_iter.py > gpurun_out/ncu_ht.log 2>&1
ls -la gpurun_out/
