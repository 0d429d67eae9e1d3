#!/bin/bash
# Run on the GPU box: resident kernel time for env variants at two Eb/N0 points of C2.
for e in "$@"; do
  echo "== $e"
  [ "$e" = "-" ] && e=""
  for pt in 0 6; do
    env $e timeout 300 python tools/prof_decode.py --config c2 --point $pt --frames 131072 --reps 2 2>&1 | grep -v "^schedule" | head -1 | sed 's/.*resident/resident/'
  done
done
