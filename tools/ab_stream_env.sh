#!/bin/bash
# Run on the GPU box: A/B library builds under one env setting.  usage: ENVS="A=1 B=2" tools/ab_stream_env.sh cfg frames point libs...
CFG=$1; F=$2; PT=$3; shift 3
for lib in "$@"; do
  echo "== $lib"
  if [ "$lib" = default ]; then L=""; else L="LDPC_LIB=$PWD/$lib"; fi
  env $L $ENVS timeout 300 python tools/prof_decode.py --config $CFG --point $PT --frames $F --reps 2 --flags ${FLAGS:-4} 2>&1 | grep -v "^schedule" | head -1 | sed -E "s/.*'check_node'/cn/; s/'syndrome.*//"
done
