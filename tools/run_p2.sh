#!/bin/bash
# ncu --set full of full-work check-node and bit-node launches (body 3, 8192 frames at the lowest Eb/N0)
O=gpurun_out/p2; mkdir -p $O
for c in c3 c4 c6; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_cn|k_bn' -s 4 -c 2 -o $O/$c \
    python tools/prof_decode.py --config $c --point 0 --frames 8192 --reps 1 > $O/${c}_prof.log 2>&1
done
ls -la $O
