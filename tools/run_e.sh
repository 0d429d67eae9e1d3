O=gpurun_out/${TAG:-r02e}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "not sanitizer" > $O/pytest_parity.log 2>&1
tail -2 $O/pytest_parity.log
for c in "c3 8192 0" "c4 8192 0" "c3 13107 2"; do
  bash tools/ab_stream.sh $c default variants/bn_g2.so variants/bn_g3.so variants/bn_g5.so variants/bn_g4m6.so >> $O/ab_bn.txt 2>&1
done
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
timeout 300 compute-sanitizer --tool synccheck tools/probe_sync > $O/probe_synccheck.log 2>&1
LDPC_NO_GRAPHS=1 timeout 600 compute-sanitizer --tool racecheck python -u tools/sanitize_run.py > $O/san_racecheck_nograph.log 2>&1; echo "racecheck nograph rc=$?" >> $O/san_rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_resident -c 1 -o $O/c2res \
    python tools/prof_decode.py --config c2 --point 2 --frames 131072 --reps 1 > $O/c2_prof.log 2>&1
python tools/ncu_summary.py $O/c2res.ncu-rep > $O/c2res_ncu_summary.txt 2>&1
python tools/ncu_lines.py $O/c2res.ncu-rep k_resident 60 > $O/c2res_lines.txt 2>&1
cat $O/san_rc.txt
