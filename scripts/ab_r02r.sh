# A/B: 64-key blocks with double-buffered S (prefill_attn.cu) vs the 128-key kernel
set -u
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_prefill_gpu.py -q -x -rf > $O/t_r02r.log 2>&1
echo "tests rc=$?"; tail -15 $O/t_r02r.log
for i in 1 2; do
  KSCD_LIB_PATH=$PWD/_exp/libkascade_pf128.so timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_r_128.txt 2>&1
  timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_r_64.txt 2>&1
done
echo pf128; cat $O/ab_r_128.txt; echo pf64; cat $O/ab_r_64.txt
