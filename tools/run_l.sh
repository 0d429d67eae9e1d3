O=gpurun_out/${TAG:-r02l}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
tail -1 $O/smoke.log
LDPC_PARITY_REPORT=$O/parity_report.jsonl timeout 2700 python -m pytest tests -q -m gpu -rf --durations=15 > $O/pytest.log 2>&1
tail -3 $O/pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
