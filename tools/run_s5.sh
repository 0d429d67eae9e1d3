#!/bin/bash
O=gpurun_out/s5; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > $O/pytest_parity.log 2>&1
tail -2 $O/pytest_parity.log
for cs in 1 2 4; do
  timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --code-streams $cs > $O/bench_c5_cs$cs.json 2> $O/bench_c5_cs$cs.err
done
