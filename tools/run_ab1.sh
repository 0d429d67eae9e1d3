#!/bin/bash
# A/B of bit-node variants (per-kernel CUDA events, plain launches): C3 and C4, 8192 frames, lowest Eb/N0
O=gpurun_out/ab1; mkdir -p $O
for c in c3 c4; do
  tools/ab_stream.sh $c 8192 0 variants/pf0.so variants/pf12.so variants/pf11.so variants/pf10.so variants/pfrv.so variants/pf0.so variants/pf12.so > $O/$c.txt 2>&1
done
cat $O/*.txt
