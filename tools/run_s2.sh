#!/bin/bash
O=gpurun_out/s2; mkdir -p $O
for c in c6 c5 c2 c4; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 300 python tools/prof_decode.py --config c6 --point 0 --frames 8192 --reps 2 --flags 4 > $O/c6_prof.txt 2>&1
