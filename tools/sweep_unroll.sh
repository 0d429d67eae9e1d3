#!/bin/bash
# Run on the GPU box: per-kernel times of the streaming sweeps for each load-batching variant.
# usage: tools/sweep_unroll.sh <config> <frames> [point]
CFG=${1:-c4}; F=${2:-8192}; PT=${3:-0}
for cu in ${CUS:-1 2 4}; do for bu in ${BUS:-1 2 3}; do
  echo "== cn_unroll=$cu bn_unroll=$bu"
  LDPC_CN_UNROLL=$cu LDPC_BN_UNROLL=$bu timeout 300 python tools/prof_decode.py --config $CFG --point $PT --frames $F --reps 2 --flags 4 2>&1 | grep -v "^schedule"
done; done
