#!/bin/bash
# global-graph resident mode: any-degree pair loop unrolled by 4 vs 1 (C6; C2 through the any-degree instance)
O=gpurun_out/ab17; mkdir -p $O
line() { timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["schedule"], d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"])'; }
for lib in gg1 gg4; do
  export LDPC_LIB=$PWD/variants/$lib.so
  echo "== c6 $lib $(line --config c6)"
  echo "== c2 generic2 $lib $(LDPC_RES_GENERIC=2 line --config c2)"
  echo "== c5 $lib $(line --config c5)"
done > $O/ab17.txt 2>&1
cat $O/ab17.txt
