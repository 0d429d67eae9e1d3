#!/bin/bash
# quick state check on one B200: smoke, C3 and C2 bench lines
O=gpurun_out/base; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err; echo "c3 rc=$?"
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err; echo "c2 rc=$?"
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c4.json 2> $O/bench_c4.err; echo "c4 rc=$?"
