#!/bin/bash
# parallel-safe variant build: tools-like but with its own tmp dir
OUT=$1; shift
D=paper_2507_10424_b200/csrc
T=$(mktemp -d)
for f in $D/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr "$@" -c $f -o $T/$(basename $f .cu).o || exit 1
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT $T/*.o
rm -rf $T
