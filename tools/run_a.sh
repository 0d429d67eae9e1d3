set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02a/smoke.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02a/bench_c3.json 2> gpurun_out/r02a/bench_c3.err
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02a/bench_c4.json 2> gpurun_out/r02a/bench_c4.err
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02a/bench_c2.json 2> gpurun_out/r02a/bench_c2.err
timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02a/bench_c5.json 2> gpurun_out/r02a/bench_c5.err
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r02a/pytest.log 2>&1
tail -3 gpurun_out/r02a/pytest.log
