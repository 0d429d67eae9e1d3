O=gpurun_out/${TAG:-r02h}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -x > $O/pytest_parity.log 2>&1
tail -2 $O/pytest_parity.log
timeout 900 python bench.py --config c6 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c6.json 2> $O/bench_c6.err
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
