#!/bin/bash
# Run on the GPU box: full ncu captures (with source) of the resident kernel (C2, 1 dB block) and of
# one k_cn / k_bn launch of the streaming schedule (C4, 1 dB block), for per-line SASS analysis.
TAG=${1:-src}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_resident -c 1 -o $OUT/res \
    python tools/prof_decode.py --config c2 --point 0 --frames 65536 --reps 1 > $OUT/res.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_cn|k_bn' -s 40 -c 2 -o $OUT/stream \
    python tools/prof_decode.py --config c4 --point 0 --frames 4096 --reps 1 --flags ${FLAGS:-0} > $OUT/stream.log 2>&1
ls -la $OUT
