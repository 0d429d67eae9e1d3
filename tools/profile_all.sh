#!/bin/bash
# Run on the GPU box: bench lines + launch lists + ncu captures for C2 (resident) and C3/C4 (streaming).
# The streaming captures skip the first launches (body 1 reads no old state): NCU_SKIP=20.
TAG=${1:-r01}
mkdir -p gpurun_out/$TAG
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$TAG/smoke.log 2>&1
NCU_COUNT=2 bash tools/profile_bench.sh $TAG/c2 c2 k_resident
NCU_COUNT=2 NCU_SKIP=20 bash tools/profile_bench.sh $TAG/c4 c4 'k_cn_pipe|k_bn'
NCU_COUNT=2 NCU_SKIP=20 bash tools/profile_bench.sh $TAG/c3 c3 'k_cn_pipe|k_bn'
for c in c2 c3 c4; do python tools/ncu_summary.py gpurun_out/$TAG/$c/full.ncu-rep > gpurun_out/$TAG/$c/ncu_summary.txt 2>&1; done
# keep the copy-back under 64 MiB: the full reports stay on the box unless KEEP_REPS=1
[ "${KEEP_REPS:-0}" = 1 ] || rm -f gpurun_out/$TAG/*/full.ncu-rep
