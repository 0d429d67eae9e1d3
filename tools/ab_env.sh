#!/bin/bash
# Run on the GPU box: per-kernel times of the streaming sweeps under different env settings.
# usage: tools/ab_env.sh <config> <frames> <point> "ENV=.. ENV2=.." "..." ...   ("-" = no extra env)
CFG=$1; F=$2; PT=$3; shift 3
for e in "$@"; do
  echo "== $e"
  [ "$e" = "-" ] && e=""
  env $e timeout 300 python tools/prof_decode.py --config $CFG --point $PT --frames $F --reps 2 --flags ${FLAGS:-4} 2>&1 | grep -v "^schedule" | head -1
done
