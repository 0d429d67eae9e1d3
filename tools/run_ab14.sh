#!/bin/bash
# BN_V8 at 12 / 14 / 16 CTAs per SM (40 / 32 / 32 registers); parity of v12
O=gpurun_out/ab14; mkdir -p $O
for c in c3 c4; do
  for lib in base v12 v14 v16 v12; do
    echo "== $c $lib"
    LDPC_LIB=$PWD/variants/$lib.so timeout 300 python tools/prof_decode.py --config $c --point 0 --frames 8192 --reps 2 --flags 6 --max-iter 10 2>&1 | grep -v "^schedule" | head -1
  done
done > $O/ab14.txt 2>&1
cat $O/ab14.txt
LDPC_LIB=$PWD/variants/v12.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > $O/parity_v12.log 2>&1; tail -1 $O/parity_v12.log
