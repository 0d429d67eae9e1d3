# v2 streaming kernels: parity on the streaming tests, then C3/C4 bench lines with and without compaction
O=gpurun_out/${TAG:-r02b}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -rf > $O/pytest_parity.log 2>&1
tail -3 $O/pytest_parity.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
LDPC_NO_COMPACT=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c3_nocompact.json 2> $O/bench_c3_nocompact.err
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
LDPC_NO_COMPACT=1 timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c4_nocompact.json 2> $O/bench_c4_nocompact.err
