# prefill softmax: exponentials against the current reference, block max only when some p > 2^8 (sum test) vs HEAD
set -u
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_prefill_gpu.py tests/test_compat_gpu.py -q -x -rf > $O/t_r02ak.log 2>&1
echo "tests rc=$?"; tail -1 $O/t_r02ak.log
for i in 1 2 3; do
  echo -n "head " >> $O/ab_ak.txt; KSCD_LIB_PATH=$PWD/_exp/libkascade_pfhead.so timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_ak.txt 2>&1
  echo -n "spec " >> $O/ab_ak.txt; timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_ak.txt 2>&1
done
cat $O/ab_ak.txt
KSCD_LIB_PATH=$PWD/_exp/libkascade_spectrace.so python scripts/pf_trace.py sparse 131072 2>&1 | head -5
KSCD_LIB_PATH=$PWD/_exp/libkascade_spectrace.so python scripts/pf_trace.py dense 32768 2>&1 | head -5
