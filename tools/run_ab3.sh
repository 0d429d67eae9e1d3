#!/bin/bash
# Bit-node timing experiments with early stop off (flags 6: every frame runs L bodies, same work per variant)
O=gpurun_out/ab3; mkdir -p $O
for c in c3 c4; do
  for lib in base xp1 xp2 base xp1; do
    echo "== $c $lib"
    LDPC_LIB=$PWD/variants/$lib.so timeout 300 python tools/prof_decode.py --config $c --point 0 --frames 8192 --reps 2 --flags 6 --max-iter 10 2>&1 | grep -v "^schedule" | head -1
  done
done > $O/ab3.txt 2>&1
cat $O/ab3.txt
