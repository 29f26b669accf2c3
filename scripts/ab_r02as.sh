# pass B fused Top-k tail on all 384 threads (registers rebalanced) vs the 256 column-sum threads
set -u
O=gpurun_out; mkdir -p $O
KSCD_LIB_PATH=$PWD/_exp/libkascade_tail384.so timeout 900 python -m pytest tests/test_prefill_gpu.py tests/test_scale_gpu.py -q -x -rf -k "prefill" > $O/t_r02as.log 2>&1
echo "variant tests rc=$?"; tail -1 $O/t_r02as.log
for i in 1 2 3; do
  echo -n "256 " >> $O/ab_as.txt; timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_as.txt 2>&1
  echo -n "384 " >> $O/ab_as.txt; KSCD_LIB_PATH=$PWD/_exp/libkascade_tail384.so timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_as.txt 2>&1
done
cat $O/ab_as.txt | sed 's/.*\(^[0-9]*\) .*"select_ms": \([0-9.]*\).*/\1 select \2/'
KSCD_LIB_PATH=$PWD/_exp/libkascade_tail384tr.so python scripts/pb_trace.py 131072 2>&1 | tail -1
