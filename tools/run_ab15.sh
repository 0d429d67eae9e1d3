#!/bin/bash
# check node with 256-bit gathers (k_cn8) at several CTA shapes vs k_cn; parity of the best candidates
O=gpurun_out/ab15; mkdir -p $O
for c in c3 c4; do
  for lib in base n2 n1 n384 n192 base n2; do
    echo "== $c $lib"
    LDPC_LIB=$PWD/variants/$lib.so timeout 300 python tools/prof_decode.py --config $c --point 0 --frames 8192 --reps 2 --flags 6 --max-iter 10 2>&1 | grep -v "^schedule" | head -1
  done
done > $O/ab15.txt 2>&1
cat $O/ab15.txt
for lib in n2 n384; do LDPC_LIB=$PWD/variants/$lib.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > $O/parity_$lib.log 2>&1; tail -1 $O/parity_$lib.log; done
