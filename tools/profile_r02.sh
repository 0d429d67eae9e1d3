#!/bin/bash
# Round-2 evidence on one B200 (run under gpurun): smoke, bench lines of every config (C3 default with the
# oracle baseline; C2 also through the generic resident instance), the launch list of the default (C3)
# bench step, ncu --set full captures of the streaming sweeps (C3, C4, C6) and the resident kernel (C2),
# their summaries / hot-SASS lists / traffic JSON, and the L2 and DRAM gather ceilings.
TAG=${1:-r02}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
for c in c4 c2 c5 c6 c1; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
LDPC_RES_GENERIC=1 timeout 900 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c2_generic.json 2> $O/bench_c2_generic.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c3_launches.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/c3_launches_bench.json 2>&1
for c in c3 c4 c6; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_cn|k_bn' -s 4 -c 2 -o $O/$c \
    python tools/prof_decode.py --config $c --point 0 --frames 8192 --reps 1 > $O/${c}_prof.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_resident -c 1 -o $O/c2res \
    python tools/prof_decode.py --config c2 --point 2 --frames 131072 --reps 1 > $O/c2_prof.log 2>&1
for r in c3 c4 c6 c2res; do
  python tools/ncu_summary.py $O/$r.ncu-rep > $O/${r}_ncu_summary.txt 2>&1
done
python tools/ncu_lines.py $O/c3.ncu-rep k_bn 30 > $O/c3_bn_hot.txt 2>&1
python tools/ncu_lines.py $O/c3.ncu-rep k_cn 30 > $O/c3_cn_hot.txt 2>&1
python tools/ncu_lines.py $O/c2res.ncu-rep k_resident 30 > $O/c2res_hot.txt 2>&1
python tools/ncu_traffic.py $O/ncu_traffic.json c3:$O/c3.ncu-rep:8192:3 c4:$O/c4.ncu-rep:8192:3 c6:$O/c6.ncu-rep:8192:3 > /dev/null 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_bw tools/l2_bw.cu 2>/dev/null
./tools/l2_bw > $O/l2_bw.json 2>&1
[ "${KEEP_REPS:-0}" = 1 ] || rm -f $O/*.ncu-rep
ls -la $O
