#!/bin/bash
# resident kernel: edge bytes (sign | isloc nibbles) vs location bytes + row-transposed sign words
O=gpurun_out/ab9; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > $O/pytest_parity.log 2>&1
tail -3 $O/pytest_parity.log
for lib in rprev reb rprev reb; do
  for c in c2 c5 c1; do
    echo "== $c $lib $(LDPC_LIB=$PWD/variants/$lib.so timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"])')"
  done
  echo "== c2g $lib $(LDPC_RES_GENERIC=1 LDPC_LIB=$PWD/variants/$lib.so timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"])')"
done > $O/ab9.txt 2>&1
cat $O/ab9.txt
