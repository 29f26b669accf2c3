set -u
O=gpurun_out; mkdir -p $O
python scripts/perf_decode_ops.py 8 32 8 131072 > $O/perf_ops_r02n.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:decode_tc_kernel' -s 0 -c 2 -o $O/dtc_r02n -f python scripts/prof_kernels.py decode > $O/dtc_ncu.out 2>&1
echo "dtc rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:topk_kernel|pool_decode' -s 0 -c 2 -o $O/sel_r02n -f python scripts/prof_kernels.py decode > $O/sel_ncu.out 2>&1
echo "sel rc=$?"
cat $O/perf_ops_r02n.txt
