O=gpurun_out/cng2; mkdir -p $O
bash tools/ab_stream.sh c6 8192 0 default variants/cng_tree0.so default variants/cng_tree0.so > $O/ab_c6.txt 2>&1
