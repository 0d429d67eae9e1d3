#!/bin/bash
# A/B of the ldpc_decode_host pipeline: buffer sets (LDPC_HOST_NBUF) and chunk size (LDPC_HOST_CHUNK_MB)
# on the C3 and C2 e2e numbers, plus its multi-chunk parity test
O=gpurun_out/host${TAG}; mkdir -p $O
if [ -n "$HOST_AB" ]; then IFS=, read -ra VARS <<< "$HOST_AB"; else VARS=("2 384" "3 384" "4 384" "3 192" "3 768"); fi
timeout 900 python -m pytest tests/test_gpu_full.py -m gpu -q -x -p no:cacheprovider -k multichunk > $O/pytest.log 2>&1; tail -n 1 $O/pytest.log
for cfg in c3 c2; do
for v in "${VARS[@]}"; do
  set -- $v
  LDPC_HOST_NBUF=$1 LDPC_HOST_CHUNK_MB=$2 timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > $O/${cfg}_nb$1_mb$2.json 2>/dev/null
done
done
