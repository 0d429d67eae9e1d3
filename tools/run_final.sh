#!/bin/bash
# the full GPU suite (with the full-batch parity report) and the round's evidence
TAG=${1:-r02}
mkdir -p gpurun_out/$TAG
rm -f gpurun_out/parity_report.jsonl
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/$TAG/pytest_gpu.log 2>&1
tail -3 gpurun_out/$TAG/pytest_gpu.log
cp gpurun_out/parity_report.jsonl gpurun_out/$TAG/parity_report.jsonl 2>/dev/null
bash tools/profile_r02.sh $TAG
