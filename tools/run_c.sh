# sanitizers with visible output, ncu captures of the v2 streaming sweeps (C3, C4), launch list of a C3 step
O=gpurun_out/${TAG:-r02c}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for tool in racecheck synccheck memcheck; do
  timeout 600 compute-sanitizer --tool $tool python tools/sanitize_run.py > $O/san_$tool.log 2>&1; echo "$tool rc=$?" >> $O/san_rc.txt
done
for c in c3 c4; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_cn|k_bn' -s 4 -c 2 -o $O/$c \
    python tools/prof_decode.py --config $c --point 0 --frames 8192 --reps 1 > $O/${c}_prof.log 2>&1
  python tools/ncu_summary.py $O/$c.ncu-rep > $O/${c}_ncu_summary.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c3_launches.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/c3_launches_bench.json 2>&1
ls -la $O
