#!/bin/bash
# usage: tools/build_variant.sh NAME "-DFOO=1 -DBAR=2"   -> build_var/lib_NAME.so (experiments only)
set -e
cd "$(dirname "$0")/../paper_1708_06290_b200/csrc"
mkdir -p /tmp/bv_$1 ../../build_var
for f in ss_api ss_sweep ss_lq ss_reduce ss_probe; do
  nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr $2 -c $f.cu -o /tmp/bv_$1/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../build_var/lib_$1.so /tmp/bv_$1/*.o -lcudart_static -lrt -ldl -lpthread
