O=gpurun_out/${TAG:-r02g}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf > $O/pytest_parity.log 2>&1
tail -2 $O/pytest_parity.log
for c in "c3 8192 0" "c4 8192 0" "c3 13107 2"; do
  bash tools/ab_stream.sh $c default variants/bn_cm0.so variants/bn_cm1g2.so variants/bn_cm0c32.so variants/bn_cm1c32.so >> $O/ab_bn.txt 2>&1
done
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
