O=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:prefill_attn_kernel<\(int\)0' -s 1 -c 1 -o $O/full_dense_prefill_r01e -f \
  python scripts/prof_kernels.py prefill 32768 > $O/full_dense_r01e.out 2>&1
echo dense rc=$?
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:pool_prefill' -s 1 -c 1 -o $O/full_pool_prefill_r01e -f \
  python scripts/prof_kernels.py prefill 32768 > $O/full_pool_r01e.out 2>&1
echo pool rc=$?
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:prefill_attn_kernel<\(int\)2' -s 1 -c 1 -o $O/full_lse_prefill_r01e -f \
  python scripts/prof_kernels.py prefill 32768 > $O/full_lse_r01e.out 2>&1
echo lse rc=$?
