#!/bin/bash
# bit node: offset records (BN_PF=3), L2 hints, 2-edge steps; early stop off (flags 6) and on (flags 4)
O=gpurun_out/ab4; mkdir -p $O
for c in c3 c4; do
  for lib in base o3 o3h o3u o3u10 o3u9 base o3; do
    echo "== $c $lib"
    LDPC_LIB=$PWD/variants/$lib.so timeout 300 python tools/prof_decode.py --config $c --point 0 --frames 8192 --reps 2 --flags 6 --max-iter 10 2>&1 | grep -v "^schedule" | head -1
  done
done > $O/ab4.txt 2>&1
cat $O/ab4.txt
