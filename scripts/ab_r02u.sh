# A/B: share of the dense / sparse prefill exponentials on the FMA-pipe polynomial (KSCD_POLY pairs per 8)
set -u
O=gpurun_out; mkdir -p $O
for i in 1 2; do
  for v in base2 poly1 poly2; do
    echo -n "$v " >> $O/ab_u.txt
    KSCD_LIB_PATH=$PWD/_exp/libkascade_$v.so timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_u.txt 2>&1
  done
done
cat $O/ab_u.txt
