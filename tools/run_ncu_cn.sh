#!/bin/bash
# ncu --set full of the C3 check node and bit node (8192 frames, every frame running), summaries + hot lines
O=gpurun_out/ncu_${1:-x}; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_cn|k_bn' -s 4 -c 2 -o $O/c3 \
    python tools/prof_decode.py --config c3 --point 0 --frames 8192 --reps 1 > $O/c3_prof.log 2>&1
python tools/ncu_summary.py $O/c3.ncu-rep > $O/c3_ncu_summary.txt 2>&1
python tools/ncu_lines.py $O/c3.ncu-rep k_cn 40 > $O/c3_cn_hot.txt 2>&1
python tools/ncu_lines.py $O/c3.ncu-rep k_bn 40 > $O/c3_bn_hot.txt 2>&1
[ "${KEEP_REPS:-0}" = 1 ] || rm -f $O/*.ncu-rep
