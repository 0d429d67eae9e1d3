O=gpurun_out/${TAG:-r02f}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for c in "c3 8192 0" "c4 8192 0" "c3 13107 2"; do
  bash tools/ab_stream.sh $c default variants/bn_g1.so variants/bn_g2.so variants/bn_g3.so variants/bn_g5.so variants/bn_g4m6.so variants/bn_g4c32.so variants/bn_g1static.so >> $O/ab_bn.txt 2>&1
done
LDPC_NO_GRAPHS=1 timeout 600 compute-sanitizer --tool synccheck python -u tools/sanitize_run.py > $O/san_synccheck_nograph.log 2>&1; echo "synccheck nograph rc=$?" >> $O/san_rc.txt
cat $O/san_rc.txt
