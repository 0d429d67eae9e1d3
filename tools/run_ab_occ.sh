#!/bin/bash
# A/B: check-node occupancy variants (per-kernel times), graph loop vs plain launches in the C3 bench
O=gpurun_out/occ; mkdir -p $O
for c in c3 c4; do
  bash tools/ab_stream.sh $c 8192 0 default variants/cn_minb4.so variants/cn_t128.so default variants/cn_minb4.so variants/cn_t128.so > $O/ab_$c.txt 2>&1
done
for rep in 1 2; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/c3_graph_$rep.json 2>/dev/null
LDPC_NO_GRAPHS=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/c3_plain_$rep.json 2>/dev/null
done
