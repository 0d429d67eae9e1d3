#!/bin/bash
# Run on the GPU box: per-kernel times of the streaming sweeps for A/B library builds.
# usage: tools/ab_stream.sh <config> <frames> <point> lib1.so lib2.so ...   ("default" = in-tree build)
CFG=$1; F=$2; PT=$3; shift 3
for lib in "$@"; do
  echo "== $lib"
  if [ "$lib" = default ]; then unset LDPC_LIB; else export LDPC_LIB=$PWD/$lib; fi
  timeout 300 python tools/prof_decode.py --config $CFG --point $PT --frames $F --reps 2 --flags 4 2>&1 | grep -v "^schedule" | head -1
done
unset LDPC_LIB
