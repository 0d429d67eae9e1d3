#!/bin/bash
# Run on the GPU box (gpurun): bench line, launch list and one full ncu capture of the top kernel.
# usage: tools/profile_bench.sh <tag> [config] [kernel-regex] [extra bench flags]
set -x
TAG=${1:-r01}; CFG=${2:-c2}; KRE=${3:-k_resident}; shift 3; EXTRA="$@"
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python bench.py --config $CFG --steps 5 --warmup 3 $EXTRA > $OUT/bench.json 2> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --config $CFG --steps 1 --warmup 0 --no-e2e --no-cpu-baseline $EXTRA > $OUT/launches_bench.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s ${NCU_SKIP:-0} -c ${NCU_COUNT:-7} -o $OUT/full \
    python bench.py --config $CFG --steps 1 --warmup 0 --no-e2e --no-cpu-baseline $EXTRA > $OUT/full_bench.log 2>&1
ls -la $OUT
