#!/bin/bash
# A/B of L2 eviction hints and the edge-ahead bit node (per-kernel CUDA events, plain launches)
O=gpurun_out/ab2; mkdir -p $O
for c in c3 c4; do
  tools/ab_stream.sh $c 8192 0 variants/base.so variants/h1.so variants/h2.so variants/h3.so variants/e2.so variants/e2h3.so variants/base.so variants/h3.so > $O/$c.txt 2>&1
  tools/ab_stream.sh $c 65536 0 variants/base.so variants/h3.so variants/e2h3.so > $O/${c}_64k.txt 2>&1
done
cat $O/*.txt
