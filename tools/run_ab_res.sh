#!/bin/bash
# A/B of the resident check-node tournament (RES_TREE): C2 bench (regular and generic instance), C5; parity
O=gpurun_out/restree; mkdir -p $O
for rep in 1 2; do
for lib in default variants/res_tree0.so; do
  if [ "$lib" = default ]; then unset LDPC_LIB; else export LDPC_LIB=$PWD/$lib; fi
  tag=$(basename $lib .so)_$rep
  timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/c2_$tag.json 2>/dev/null
  LDPC_RES_GENERIC=1 timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/c2g_$tag.json 2>/dev/null
done
done
unset LDPC_LIB
timeout 600 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5.json 2>/dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "not sanitizer" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 900 python -m pytest tests/test_gpu_full.py -m gpu -q -x -p no:cacheprovider -k "c1 or c2 or c5" > $O/pytest_full.log 2>&1; tail -2 $O/pytest_full.log
