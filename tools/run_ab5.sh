#!/bin/bash
# check node: paired edge update (CN_PAIR) vs edge-by-edge; then the parity suite on the in-tree build
O=gpurun_out/ab5; mkdir -p $O
for c in c3 c4; do
  for lib in base pair base pair; do
    echo "== $c $lib"
    LDPC_LIB=$PWD/variants/$lib.so timeout 300 python tools/prof_decode.py --config $c --point 0 --frames 8192 --reps 2 --flags 6 --max-iter 10 2>&1 | grep -v "^schedule" | head -1
  done
done > $O/ab5.txt 2>&1
cat $O/ab5.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > $O/pytest_parity.log 2>&1
tail -3 $O/pytest_parity.log
