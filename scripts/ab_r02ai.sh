# sparse prefill: tree max (8 FMNMX3 chains) vs the serial running max
set -u
O=gpurun_out; mkdir -p $O
for i in 1 2 3; do
  echo -n "serial " >> $O/ab_ai.txt; timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_ai.txt 2>&1
  echo -n "tree " >> $O/ab_ai.txt; KSCD_LIB_PATH=$PWD/_exp/libkascade_tree.so timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_ai.txt 2>&1
done
cat $O/ab_ai.txt | sed 's/"dense_ms.*"sparse_ms"/ ... "sparse_ms"/'
KSCD_LIB_PATH=$PWD/_exp/libkascade_treetrace.so python scripts/pf_trace.py sparse 131072 2>&1 | head -8
