set -u
O=gpurun_out; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:prefill_attn_kernel<\(int\)1' -s 1 -c 1 -o $O/sp_r02s -f python scripts/prof_kernels.py prefill 131072 > $O/sp_ncu.out 2>&1
echo "sp rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:prefill_attn_kernel<\(int\)0' -s 1 -c 1 -o $O/dn_r02s -f python scripts/prof_kernels.py prefill 32768 > $O/dn_ncu.out 2>&1
echo "dn rc=$?"
