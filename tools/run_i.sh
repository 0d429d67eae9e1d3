O=gpurun_out/${TAG:-r02i}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -x -k "not sanitizer" > $O/pytest_parity.log 2>&1
tail -2 $O/pytest_parity.log
timeout 900 python bench.py --config c6 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c6.json 2> $O/bench_c6.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_cn|k_bn' -s 4 -c 2 -o $O/c6 \
    python tools/prof_decode.py --config c6 --point 0 --frames 8192 --reps 1 > $O/c6_prof.log 2>&1
python tools/ncu_summary.py $O/c6.ncu-rep > $O/c6_ncu_summary.txt 2>&1
python tools/ncu_lines.py $O/c6.ncu-rep k_cn 25 > $O/c6_cn_hot.txt 2>&1
rm -f $O/*.ncu-rep
