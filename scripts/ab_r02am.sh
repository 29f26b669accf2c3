# sparse prefill: share of key pairs on the degree-3 FMA exp2 polynomial (KSCD_SPARSE_POLY3 per 8)
set -u
O=gpurun_out; mkdir -p $O
for i in 1 2; do
  echo -n "p3_0 " >> $O/ab_am.txt; timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_am.txt 2>&1
  for v in p3_1 p3_2 p3_3; do
    echo -n "$v " >> $O/ab_am.txt; KSCD_LIB_PATH=$PWD/_exp/libkascade_$v.so timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_am.txt 2>&1
  done
done
cat $O/ab_am.txt | sed 's/.*\(p3_[0-9]\).*"sparse_ms": \([0-9.]*\).*/\1 \2/'
KSCD_LIB_PATH=$PWD/_exp/libkascade_p3_2.so timeout 900 python -m pytest tests/test_prefill_gpu.py tests/test_compat_gpu.py -q -rf 2>&1 | tail -3
