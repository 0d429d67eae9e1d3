O=gpurun_out/${TAG:-r02d}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "not sanitizer" > $O/pytest_parity.log 2>&1
tail -2 $O/pytest_parity.log
for tool in memcheck synccheck racecheck; do
  timeout 600 compute-sanitizer --tool $tool python -u tools/sanitize_run.py > $O/san_$tool.log 2>&1; echo "$tool rc=$?" >> $O/san_rc.txt
done
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
for c in c3 c4; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_cn|k_bn' -s 4 -c 2 -o $O/$c \
    python tools/prof_decode.py --config $c --point 0 --frames 8192 --reps 1 > $O/${c}_prof.log 2>&1
  python tools/ncu_summary.py $O/$c.ncu-rep > $O/${c}_ncu_summary.txt 2>&1
done
cat $O/san_rc.txt
