#!/bin/bash
# build an experimental variant of libhj.so with extra nvcc defines into $1 (e.g. /tmp/libhj_v.so)
out=$1; shift
mkdir -p /tmp/hjvar_$(basename $out .so)
objs=""
for f in paper_1405_3521_b200/csrc/*.cu; do
  o=/tmp/hjvar_$(basename $out .so)/$(basename $f).o
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr "$@" -c $f -o $o &
  objs="$objs $o"
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $out $objs -lcudart
