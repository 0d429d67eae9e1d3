#!/bin/bash
# resident: bounded-degree (<= 8) instance as the generic one; parity; C2 lines of each instance
O=gpurun_out/ab10; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > $O/pytest_parity.log 2>&1
tail -3 $O/pytest_parity.log
line() { timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"])'; }
for lib in reb rb8; do
  export LDPC_LIB=$PWD/variants/$lib.so
  echo "== c2 $lib regular $(line)"
  echo "== c2 $lib generic1 $(LDPC_RES_GENERIC=1 line)"
  echo "== c2 $lib generic2 $(LDPC_RES_GENERIC=2 line)"
done > $O/ab10.txt 2>&1
cat $O/ab10.txt
