# sparse prefill: ex2.approx.f16x2 (two exponentials per MUFU op) vs fp32 MUFU exponentials; parity tests on the variant
set -u
O=gpurun_out; mkdir -p $O
for i in 1 2 3; do
  echo -n "f32 " >> $O/ab_aj.txt; timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_aj.txt 2>&1
  echo -n "f16 " >> $O/ab_aj.txt; KSCD_LIB_PATH=$PWD/_exp/libkascade_f16exp.so timeout 300 python scripts/perf_prefill.py 131072 >> $O/ab_aj.txt 2>&1
done
cat $O/ab_aj.txt | sed 's/"dense_ms.*"sparse_ms"/ ... "sparse_ms"/'
KSCD_LIB_PATH=$PWD/_exp/libkascade_f16trace.so python scripts/pf_trace.py sparse 131072 2>&1 | head -4
KSCD_LIB_PATH=$PWD/_exp/libkascade_f16exp.so timeout 1500 python -m pytest tests/test_prefill_gpu.py tests/test_scale_gpu.py tests/test_compat_gpu.py tests/test_exporter_traces_gpu.py tests/test_cli_gpu.py tests/test_acceptance_gpu.py -q -rf -k "prefill or compat or exporter or cli or acceptance or trace" > $O/t_r02aj.log 2>&1
echo "variant tests rc=$?"; grep -E "passed|failed|FAILED|Error" $O/t_r02aj.log | tail -12
