#!/bin/bash
# Build an A/B variant of libideq.so with extra nvcc defines for conv_tc.cu only:
#   tools/build_variant.sh NAME -DFOO=1 ...   ->  paper_2605_19705_b200/lib/variants/libideq_NAME.so
# (select it at run time with IDEQ_LIB=<path>; the default build is untouched)
set -e
cd "$(dirname "$0")/.."
python -m paper_2605_19705_b200.build >/dev/null
name=$1; shift
L=paper_2605_19705_b200/lib
mkdir -p $L/variants/$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  --expt-relaxed-constexpr -diag-suppress 177,128 -I include "$@" -c paper_2605_19705_b200/csrc/conv_tc.cu -o $L/variants/$name/conv_tc.o
objs=$(ls $L/obj/*.o | grep -v '/conv_tc.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $L/variants/libideq_$name.so $objs $L/variants/$name/conv_tc.o \
  -cudart static -ldl -lpthread -lrt
echo $L/variants/libideq_$name.so
