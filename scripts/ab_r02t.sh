# A/B: pipelined TMEM loads + speculative exponentials (dense/sparse prefill) vs base
set -u
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_prefill_gpu.py -q -x -rf > $O/t_r02t.log 2>&1
echo "tests rc=$?"; tail -3 $O/t_r02t.log
for i in 1 2; do
  KSCD_LIB_PATH=$PWD/_exp/libkascade_base.so timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_t_base.txt 2>&1
  timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_t_new.txt 2>&1
done
echo base; cat $O/ab_t_base.txt; echo new; cat $O/ab_t_new.txt
