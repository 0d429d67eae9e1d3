O=gpurun_out/${TAG:-r02k}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
LDPC_CN_BULK=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -rf -x -k "stream_variants or high_degree or c6 or randomised or compaction or signed" > $O/pytest_bulk.log 2>&1
tail -3 $O/pytest_bulk.log
for c in "c3 8192 0" "c4 8192 0" "c6 8192 0" "c3 13107 2"; do
  bash tools/ab_env.sh $c - LDPC_CN_BULK=1 >> $O/ab_bulk.txt 2>&1
done
LDPC_CN_BULK=1 timeout 900 python bench.py --config c6 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c6_bulk.json 2> $O/bench_c6_bulk.err
