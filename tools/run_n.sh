O=gpurun_out/${TAG:-r02n}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for c in "c3 8192 0" "c4 8192 0" "c3 13107 2"; do
  bash tools/ab_stream.sh $c default variants/cn_pf.so variants/cn_pf_smemu.so >> $O/ab_cn.txt 2>&1
done
