#!/bin/bash
# Run on the GPU box: ncu --set full captures for the roofline "traffic" fields.
#  c2: the single resident launch of one bench step (whole batch);
#  c3/c4: with --per-block, launches 21-22 of the streaming kernels fall in the first Eb/N0 block
#         (every frame running), whose algorithmic bytes are known exactly.
OUT=gpurun_out/caps; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_resident -c 1 -o $OUT/c2 \
    python bench.py --config c2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for c in c3 c4; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_cn_pipe|k_bn' -s 20 -c 2 -o $OUT/$c \
      python bench.py --config $c --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --per-block > /dev/null 2>&1
done
for c in c2 c3 c4; do python tools/ncu_summary.py $OUT/$c.ncu-rep > $OUT/${c}_summary.txt 2>&1; rm -f $OUT/$c.ncu-rep; done
