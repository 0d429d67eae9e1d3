#!/bin/bash
# Run on the GPU box: per-kernel times of the streaming sweeps with and without environment knobs.
# usage: tools/ab_env.sh <config> <frames> <point> "ENV=1" "ENV2=1 ENV3=0" ...   ("-" = no knob)
CFG=$1; F=$2; PT=$3; shift 3
for e in "$@"; do
  echo "== $e"
  if [ "$e" = "-" ]; then e=""; fi
  env $e timeout 300 python tools/prof_decode.py --config $CFG --point $PT --frames $F --reps 2 --flags 4 2>&1 | grep -v "^schedule" | head -1
done
