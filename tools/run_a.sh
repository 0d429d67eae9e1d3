# round-2 GPU pass: smoke, default bench line, the GPU test suite, the other configs' bench lines
O=gpurun_out/${TAG:-r02a}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 2700 python -m pytest tests -q -m gpu -rf --durations=30 > $O/pytest.log 2>&1
for c in c4 c2 c5; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
tail -5 $O/pytest.log
