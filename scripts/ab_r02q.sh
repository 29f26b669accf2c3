# A/B: softmax warpgroups take turns on the MUFU (KSCD_PF_TOKEN) vs not
set -u
O=gpurun_out; mkdir -p $O
for i in 1 2; do
  KSCD_LIB_PATH=$PWD/_exp/libkascade_notoken.so python scripts/perf_prefill.py 131072 >> $O/ab_q_notoken.txt 2>&1
  python scripts/perf_prefill.py 131072 >> $O/ab_q_token.txt 2>&1
done
echo notoken; cat $O/ab_q_notoken.txt; echo token; cat $O/ab_q_token.txt
timeout 1200 python -m pytest tests/test_prefill_gpu.py -q -x -rf > $O/t_r02q.log 2>&1
echo "tests rc=$?"; tail -3 $O/t_r02q.log
