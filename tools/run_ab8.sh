#!/bin/bash
# any-degree check node (C6, d = 32): edge pairs vs edge by edge; C6 bench; parity
O=gpurun_out/ab8; mkdir -p $O
for lib in np p np p; do
  echo "== c6 $lib"
  LDPC_LIB=$PWD/variants/$lib.so timeout 300 python tools/prof_decode.py --config c6 --point 0 --frames 8192 --reps 2 --flags 6 --max-iter 12 2>&1 | grep -v "^schedule" | head -1
done > $O/ab8.txt 2>&1
for lib in np p; do
  echo "== c6bench $lib $(LDPC_LIB=$PWD/variants/$lib.so timeout 600 python bench.py --config c6 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"])')" >> $O/ab8.txt
done
cat $O/ab8.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > $O/pytest_parity.log 2>&1
tail -3 $O/pytest_parity.log
