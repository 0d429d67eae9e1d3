#!/bin/bash
# check node: eta^prev by integer multiply-adds on the FMA pipe (CN_FMASEL) vs FSEL/LOP3 on the ALU pipe
O=gpurun_out/ab20; mkdir -p $O
for c in c3 c4; do
  for lib in cbase cfma cbase cfma; do
    echo "== $c $lib"
    LDPC_LIB=$PWD/variants/$lib.so timeout 300 python tools/prof_decode.py --config $c --point 0 --frames 8192 --reps 2 --flags 6 --max-iter 10 2>&1 | grep -v "^schedule" | head -1
  done
done
line() { timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"], d["clocks"].get("power_w_median"), {k:v["avg_launch_us"] for k,v in (r.get("sweeps") or {}).items()})'; }
for lib in cbase cfma cbase cfma; do
  export LDPC_LIB=$PWD/variants/$lib.so
  echo "== bench c3 $lib $(line --config c3)"
done
LDPC_LIB=$PWD/variants/cfma.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > $O/parity.log 2>&1; tail -1 $O/parity.log
