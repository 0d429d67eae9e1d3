#!/bin/bash
# Per-kernel A/B of one variant library against the in-tree build (C3, C4, C6; 8192 frames, every frame
# running), its stream parity tests, and the C3 bench line of both.  usage: tools/ab_variant.sh variants/x.so
V=$1; T=$(basename $V .so); O=gpurun_out/ab_$T; mkdir -p $O
for c in c3 c4 c6; do bash tools/ab_stream.sh $c 8192 0 default $V default $V > $O/ab_$c.txt 2>&1; done
LDPC_LIB=$PWD/$V timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "not sanitizer" > $O/pytest.log 2>&1; tail -n 1 $O/pytest.log
LDPC_LIB=$PWD/$V timeout 900 python -m pytest tests/test_gpu_full.py -m gpu -q -x -p no:cacheprovider -k "c3 or c4" > $O/pytest_full.log 2>&1; tail -n 1 $O/pytest_full.log
LDPC_LIB=$PWD/$V timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/c3_variant.json 2>/dev/null
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/c3_default.json 2>/dev/null
