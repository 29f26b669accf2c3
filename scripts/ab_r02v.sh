# A/B: two softmax warps per (tile, lane quarter), 64 keys each (KSCD_PF_SPLIT=2) vs base
set -u
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_prefill_gpu.py -q -x -rf > $O/t_r02v.log 2>&1
echo "tests rc=$?"; tail -3 $O/t_r02v.log
for i in 1 2; do
  echo -n "base " >> $O/ab_v.txt; KSCD_LIB_PATH=$PWD/_exp/libkascade_base2.so timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_v.txt 2>&1
  echo -n "split " >> $O/ab_v.txt; timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_v.txt 2>&1
done
cat $O/ab_v.txt
