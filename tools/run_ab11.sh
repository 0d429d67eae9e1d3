#!/bin/bash
# check node: L2 eviction hints (bit 0: row records evict_first; bit 1: s gathers evict_last)
O=gpurun_out/ab11; mkdir -p $O
for c in c4 c3; do
  for lib in c0 c1 c2 c3 c0 c1 c2 c3; do
    echo "== $c $lib"
    LDPC_LIB=$PWD/variants/$lib.so timeout 300 python tools/prof_decode.py --config $c --point 0 --frames 8192 --reps 2 --flags 6 --max-iter 10 2>&1 | grep -v "^schedule" | head -1
  done
done > $O/ab11.txt 2>&1
cat $O/ab11.txt
