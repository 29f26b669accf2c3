# dense / sparse prefill: S in two 64-key halves with parity-alternating TMEM columns (first half of S(j+1)
# issued during softmax(j)) vs HEAD
set -u
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_prefill_gpu.py tests/test_compat_gpu.py -q -x -rf > $O/t_r02ao.log 2>&1
echo "tests rc=$?"; tail -3 $O/t_r02ao.log
for i in 1 2 3; do
  echo -n "head " >> $O/ab_ao.txt; KSCD_LIB_PATH=$PWD/_exp/libkascade_pfhead.so timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_ao.txt 2>&1
  echo -n "split " >> $O/ab_ao.txt; timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_ao.txt 2>&1
done
cat $O/ab_ao.txt | sed 's/"select_ms[^,]*, //; s/"lse_pass_tflops[^,]*, //; s/"dense_tflops[^,]*, //; s/"N": 131072, //'
KSCD_LIB_PATH=$PWD/_exp/libkascade_splittrace.so python scripts/pf_trace.py dense 32768 2>&1 | head -9
KSCD_LIB_PATH=$PWD/_exp/libkascade_splittrace.so python scripts/pf_trace.py sparse 131072 2>&1 | head -4
