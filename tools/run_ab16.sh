#!/bin/bash
# C6 on the resident schedule with the edge lists in global memory vs the streaming schedule; parity
O=gpurun_out/ab16; mkdir -p $O
export LDPC_LIB=$PWD/variants/gg.so
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "c6 or global_graph or c5 or c2_subset or generic" > $O/pytest.log 2>&1
tail -2 $O/pytest.log
line() { timeout 900 python bench.py --config c6 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["schedule"], d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"])'; }
echo "== c6 default (gg) $(line)"
echo "== c6 stream $(line --flags 4)"
echo "== c6 gg S=8 $(LDPC_RES_SLOTS=8 line)"
