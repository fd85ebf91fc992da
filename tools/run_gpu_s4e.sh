# ncu --set full of the encoder/decoder conv launches (IDs 4..29) and the first VJP launches (36..38) of one eager C3 iteration
mkdir -p gpurun_out/s4e
timeout 900 ncu -f --set full --import-source on --clock-control none --launch-skip 4 --launch-count 26 \
  -o gpurun_out/s4e/convs python tools/one_iter.py > gpurun_out/s4e/ncu.log 2>&1; echo full $?
ncu -i gpurun_out/s4e/convs.ncu-rep --page raw --csv > gpurun_out/s4e/convs_raw.csv 2>/dev/null
ncu -i gpurun_out/s4e/convs.ncu-rep --page details > gpurun_out/s4e/convs_details.txt 2>/dev/null
rm -f gpurun_out/s4e/convs.ncu-rep
wc -l gpurun_out/s4e/*
