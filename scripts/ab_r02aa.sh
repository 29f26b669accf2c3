# decode Top-k shape: 512-thread CTAs x 4-CTA clusters (0) vs 256 x 8 (1), 256 x 4 (2), 128 x 8 (3)
set -u
O=gpurun_out; mkdir -p $O
for i in 1 2; do
  for v in tk1 tk2 tk3; do
    echo "== $v" >> $O/ab_aa.txt; KSCD_LIB_PATH=$PWD/_exp/libkascade_$v.so python scripts/perf_decode_ops.py 8 32 8 131072 2>&1 | grep -E "select" >> $O/ab_aa.txt
  done
  echo "== tk0" >> $O/ab_aa.txt; python scripts/perf_decode_ops.py 8 32 8 131072 2>&1 | grep -E "select" >> $O/ab_aa.txt
done
cat $O/ab_aa.txt
KSCD_LIB_PATH=$PWD/_exp/libkascade_tk1.so timeout 600 python -m pytest tests/test_decode_gpu.py -q -x -k "topk or select" 2>&1 | tail -2
