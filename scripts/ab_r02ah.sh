# dense prefill: K half-stages freed by S retire (own k_empty + V producer thread) vs HEAD; per-block traces
set -u
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_prefill_gpu.py -q -x -rf > $O/t_r02ah.log 2>&1
echo "tests rc=$?"; tail -1 $O/t_r02ah.log
for i in 1 2; do
  echo -n "base " >> $O/ab_ah.txt; KSCD_LIB_PATH=$PWD/_exp/libkascade_pfbase.so timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_ah.txt 2>&1
  echo -n "kfree " >> $O/ab_ah.txt; timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_ah.txt 2>&1
done
cat $O/ab_ah.txt
echo "== trace HEAD sparse"; KSCD_LIB_PATH=$PWD/_exp/libkascade_pftrace0.so python scripts/pf_trace.py sparse 131072 2>&1 | head -9
echo "== trace new dense"; KSCD_LIB_PATH=$PWD/_exp/libkascade_pftrace.so python scripts/pf_trace.py dense 32768 2>&1 | head -9
