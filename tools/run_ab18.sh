#!/bin/bash
# resident kernel: slots per CTA / CTA size on C2 and C5 (planner default: C2 S=8 x 2 CTAs of 256, C5 S=4 compact)
O=gpurun_out/ab18; mkdir -p $O
line() { timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])'; }
echo "== c2 default $(line --config c2)"
echo "== c2 S16 $(LDPC_RES_SLOTS=16 line --config c2)"
echo "== c2 S4 $(LDPC_RES_SLOTS=4 line --config c2)"
echo "== c2 S8 T512 $(LDPC_RES_SLOTS=8 LDPC_RES_THREADS=512 line --config c2)"
echo "== c2 S8 T128 $(LDPC_RES_SLOTS=8 LDPC_RES_THREADS=128 line --config c2)"
echo "== c2 S16 T1024 $(LDPC_RES_SLOTS=16 LDPC_RES_THREADS=1024 line --config c2)"
echo "== c5 default $(line --config c5)"
echo "== c5 T256 $(LDPC_RES_THREADS=256 line --config c5)"
