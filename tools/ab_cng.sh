O=gpurun_out/cng3; mkdir -p $O
bash tools/ab_stream.sh c6 8192 0 default variants/cng_tree0.so default variants/cng_tree0.so > $O/ab_c6.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "not sanitizer" > $O/pytest.log 2>&1; tail -n 1 $O/pytest.log
timeout 900 python -m pytest tests/test_gpu_full.py -m gpu -q -x -p no:cacheprovider -k "c6 or dense" > $O/pytest_full.log 2>&1; tail -n 1 $O/pytest_full.log
timeout 600 python bench.py --config c6 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/c6.json 2>/dev/null
