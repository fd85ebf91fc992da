# conv_tc bisection: per-layer ncu times of one eager C3 iteration with parts of the kernel switched off
set -x
mkdir -p gpurun_out/s2j
timeout 300 python tools/one_iter.py > gpurun_out/s2j/plain.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv_tc --csv --log-file gpurun_out/s2j/base.csv python tools/one_iter.py > /dev/null 2>&1; echo base $?
for v in noepi nob noa noab noall; do IDEQ_LIB=paper_2605_19705_b200/lib/variants/libideq_$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv_tc --csv --log-file gpurun_out/s2j/$v.csv python tools/one_iter.py > gpurun_out/s2j/$v.log 2>&1; echo $v $?; done
