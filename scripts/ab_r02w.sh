# A/B: one MMA issuer per tile in the dense prefill (KSCD_PF_2MMA) vs one shared issuer
set -u
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_prefill_gpu.py -q -x -rf > $O/t_r02w.log 2>&1
echo "tests rc=$?"; tail -2 $O/t_r02w.log
for i in 1 2; do
  echo -n "one " >> $O/ab_w.txt; KSCD_LIB_PATH=$PWD/_exp/libkascade_one_mma.so timeout 300 python scripts/perf_prefill.py 131072 dense-only >> $O/ab_w.txt 2>&1
  echo -n "two " >> $O/ab_w.txt; timeout 300 python scripts/perf_prefill.py 131072 dense-only >> $O/ab_w.txt 2>&1
done
cat $O/ab_w.txt
