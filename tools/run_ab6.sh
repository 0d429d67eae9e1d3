#!/bin/bash
# bit node: cp.async stages (BN_PF=4, BN_NB edges in flight per warp) vs offset-record loads; parity of one
O=gpurun_out/ab6; mkdir -p $O
for c in c3 c4; do
  for lib in base a3 a4 a6 a8 base; do
    echo "== $c $lib"
    LDPC_LIB=$PWD/variants/$lib.so timeout 300 python tools/prof_decode.py --config $c --point 0 --frames 8192 --reps 2 --flags 6 --max-iter 10 2>&1 | grep -v "^schedule" | head -1
  done
done > $O/ab6.txt 2>&1
cat $O/ab6.txt
for lib in a4 a6; do LDPC_LIB=$PWD/variants/$lib.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "stream or c3 or c4 or random or compaction" > $O/parity_$lib.log 2>&1; tail -2 $O/parity_$lib.log; done
