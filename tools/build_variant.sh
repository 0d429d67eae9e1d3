#!/bin/bash
# Build an A/B variant of libldpc.so with extra nvcc defines: tools/build_variant.sh <out.so> -DFOO=1 ...
OUT=$1; shift
D=paper_2507_10424_b200/csrc
mkdir -p /tmp/ldpcv
for f in $D/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr "$@" -c $f -o /tmp/ldpcv/$(basename $f .cu).o || exit 1
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT /tmp/ldpcv/*.o
