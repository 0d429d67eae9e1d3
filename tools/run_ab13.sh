#!/bin/bash
# bit node with 256-bit accesses (BN_V8) at 12 / 10 / 8 CTAs per SM vs the float4 bit node; parity of each
O=gpurun_out/ab13; mkdir -p $O
for c in c3 c4 c6; do
  for lib in base v12 v10 v8 base v10; do
    echo "== $c $lib"
    LDPC_LIB=$PWD/variants/$lib.so timeout 300 python tools/prof_decode.py --config $c --point 0 --frames 8192 --reps 2 --flags 6 --max-iter 10 2>&1 | grep -v "^schedule" | head -1
  done
done > $O/ab13.txt 2>&1
cat $O/ab13.txt
for lib in v10 v8; do LDPC_LIB=$PWD/variants/$lib.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > $O/parity_$lib.log 2>&1; tail -1 $O/parity_$lib.log; done
