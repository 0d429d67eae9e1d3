O=gpurun_out/${TAG:-r02o}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -x -k "binding or counters" > $O/pytest_new.log 2>&1
tail -3 $O/pytest_new.log
for c in "c6 8192 0" "c6 8192 3"; do
  bash tools/ab_stream.sh $c default variants/cng_pf.so >> $O/ab_cng.txt 2>&1
done
