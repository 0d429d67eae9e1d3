#!/bin/bash
O=gpurun_out/p1; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_resident -c 1 -o $O/c2res \
    python tools/prof_decode.py --config c2 --point 2 --frames 65536 --reps 1 > $O/c2_prof.log 2>&1
ls -la $O
