#!/bin/bash
# A/B of the check-node tournament (CN_TREE) + stream parity tests + C3/C4 bench lines
O=gpurun_out/tree; mkdir -p $O
for c in c3 c4; do
  bash tools/ab_stream.sh $c 8192 0 default variants/cn_tree0.so default variants/cn_tree0.so > $O/ab_$c.txt 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "not sanitizer" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 900 python -m pytest tests/test_gpu_full.py -m gpu -q -x -p no:cacheprovider -k "c3 or c4 or c6" > $O/pytest_full.log 2>&1; tail -2 $O/pytest_full.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c4.json 2> $O/bench_c4.err
