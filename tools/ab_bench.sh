#!/bin/bash
# Whole-step A/B of variant libraries on bench lines (alternating, REPS rounds).
# usage: CFGS="c3 c4" REPS=2 tools/ab_bench.sh default variants/a.so variants/b.so
O=gpurun_out/abb${TAG}; mkdir -p $O
for rep in $(seq ${REPS:-2}); do
for cfg in ${CFGS:-c3}; do
for lib in "$@"; do
  if [ "$lib" = default ]; then unset LDPC_LIB; else export LDPC_LIB=$PWD/$lib; fi
  timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/${cfg}_$(basename $lib .so)_$rep.json 2>/dev/null
done; done; done
unset LDPC_LIB
