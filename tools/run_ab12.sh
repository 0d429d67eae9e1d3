#!/bin/bash
# whole-bench A/B on one box: previous build (cur) vs check-node pairs off + packed resident records (new)
O=gpurun_out/ab12; mkdir -p $O
line() { timeout 600 python bench.py --config $1 --steps $2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"], d["clocks"].get("power_w_median"), {k:v["avg_launch_us"] for k,v in (r.get("sweeps") or {}).items()})'; }
for rep in 1 2; do
  for lib in cur new; do
    export LDPC_LIB=$PWD/variants/$lib.so
    for c in c3 c2 c5; do echo "== $c $lib $(line $c 5)"; done
  done
done > $O/ab12.txt 2>&1
cat $O/ab12.txt
