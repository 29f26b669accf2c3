# dense / sparse prefill softmax: FMA-pipe polynomial share (KSCD_POLY pairs per 8) on the speculative softmax
set -u
O=gpurun_out; mkdir -p $O
for i in 1 2; do
  echo -n "poly0 " >> $O/ab_al.txt; timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_al.txt 2>&1
  for v in poly1 poly2; do
    echo -n "$v " >> $O/ab_al.txt; KSCD_LIB_PATH=$PWD/_exp/libkascade_$v.so timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_al.txt 2>&1
  done
done
cat $O/ab_al.txt | sed 's/"select_ms[^,]*, //; s/"lse_pass_tflops[^,]*, //; s/"dense_tflops[^,]*, //'
