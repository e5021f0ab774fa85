#!/bin/bash
# build_variant.sh NAME "-DFOO=1 ..."  -> build_var/NAME/libcbfs.so (performance experiments)
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
OUT=build_var/$NAME; mkdir -p $OUT
for f in graph cbfs sparse select query labels pll digest; do
  nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC $@ -c paper_2410_17226_b200/csrc/$f.cu -o $OUT/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libcbfs.so $OUT/*.o -lcudart
echo built $OUT/libcbfs.so
