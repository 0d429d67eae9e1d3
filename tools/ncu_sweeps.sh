#!/bin/bash
# Run on the GPU box: ncu --set full of one config's streaming sweeps (8192 frames of the lowest Eb/N0
# block, every frame running; launches 5-6 = body 3's check node and bit node), summary and hot SASS lines.
# usage: tools/ncu_sweeps.sh <tag> [config]      (KEEP_REPS=1 keeps the .ncu-rep)
TAG=${1:-x}; CFG=${2:-c3}
O=gpurun_out/ncu_$TAG; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_cn|k_bn' -s 4 -c 2 -o $O/$CFG \
    python tools/prof_decode.py --config $CFG --point 0 --frames 8192 --reps 1 > $O/${CFG}_prof.log 2>&1
python tools/ncu_summary.py $O/$CFG.ncu-rep > $O/${CFG}_ncu_summary.txt 2>&1
python tools/ncu_lines.py $O/$CFG.ncu-rep k_cn 40 > $O/${CFG}_cn_hot.txt 2>&1
python tools/ncu_lines.py $O/$CFG.ncu-rep k_bn 40 > $O/${CFG}_bn_hot.txt 2>&1
[ "${KEEP_REPS:-0}" = 1 ] || rm -f $O/*.ncu-rep
