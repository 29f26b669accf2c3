# prefill softmax: S in two TMEM-load halves overlapped with the speculative exponentials vs HEAD
set -u
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_prefill_gpu.py tests/test_compat_gpu.py -q -x -rf > $O/t_r02an.log 2>&1
echo "tests rc=$?"; tail -1 $O/t_r02an.log
for i in 1 2 3; do
  echo -n "head " >> $O/ab_an.txt; KSCD_LIB_PATH=$PWD/_exp/libkascade_pfhead.so timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_an.txt 2>&1
  echo -n "halves " >> $O/ab_an.txt; timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_an.txt 2>&1
done
cat $O/ab_an.txt | sed 's/"select_ms[^,]*, //; s/"lse_pass_tflops[^,]*, //; s/"dense_tflops[^,]*, //; s/"N": 131072, //'
