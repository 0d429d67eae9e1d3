#!/bin/bash
# resident: global loads of the D sweep issued first (early) vs after the outputs (prev)
O=gpurun_out/ab19; mkdir -p $O
line() { timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])'; }
for lib in prev early prev early; do
  export LDPC_LIB=$PWD/variants/$lib.so
  echo "== c2 $lib $(line --config c2)"
  echo "== c5 $lib $(line --config c5)"
  echo "== c2g $lib $(LDPC_RES_GENERIC=1 line --config c2)"
done
LDPC_LIB=$PWD/variants/early.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > $O/parity.log 2>&1; tail -1 $O/parity.log
