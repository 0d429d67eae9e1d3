#!/bin/bash
# e2e of one config under host-pipeline settings.  usage: CFG=c6 HOST_AB="2 384,3 384,3 768,3 1536" tools/ab_host_cfg.sh
O=gpurun_out/hostcfg; mkdir -p $O
IFS=, read -ra VARS <<< "$HOST_AB"
for cfg in $CFG; do
for v in "${VARS[@]}"; do
  set -- $v
  LDPC_HOST_NBUF=$1 LDPC_HOST_CHUNK_MB=$2 timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > $O/${cfg}_nb$1_mb$2.json 2>/dev/null
done
done
