# A/B: speculative-reference prefill softmax vs base; engine launch merging
set -u
O=gpurun_out; mkdir -p $O
for i in 1 2; do
  KSCD_LIB_PATH=$PWD/_exp/libkascade_base.so python scripts/perf_prefill.py 131072 >> $O/ab_prefill_base.txt 2>&1
  python scripts/perf_prefill.py 131072 >> $O/ab_prefill_new.txt 2>&1
done
echo base; cat $O/ab_prefill_base.txt; echo new; cat $O/ab_prefill_new.txt
timeout 1200 python -m pytest tests/test_prefill_gpu.py tests/test_decode_gpu.py tests/test_scale_gpu.py -q -x -rf > $O/t_r02o.log 2>&1
echo "tests rc=$?"; tail -3 $O/t_r02o.log
timeout 900 python bench.py --no-prefill --no-cpu-baseline --no-configs --no-parity-sample > $O/bench_dec_r02o.json 2>$O/bench_dec_r02o.err
echo "bench rc=$?"; python -c "
import json;d=json.loads(open('$O/bench_dec_r02o.json').read().strip().splitlines()[-1]);print(d['value'],d['dense_us_per_token'],d['gpu_launches'],d['e2e']['value'])"
