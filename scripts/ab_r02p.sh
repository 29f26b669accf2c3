# fused decode pooling (Top-k first pass) check + timing
set -u
O=gpurun_out; mkdir -p $O
python scripts/perf_decode_ops.py 8 32 8 131072 > $O/perf_ops_r02p.txt 2>&1; cat $O/perf_ops_r02p.txt
python scripts/perf_decode_ops.py 8 8 1 131072 >> $O/perf_ops_r02p.txt 2>&1; tail -6 $O/perf_ops_r02p.txt
timeout 1200 python -m pytest tests/test_decode_gpu.py tests/test_scale_gpu.py tests/test_pre_pooling_gpu.py tests/test_sharding_gpu.py -q -x -rf > $O/t_r02p.log 2>&1
echo "tests rc=$?"; tail -3 $O/t_r02p.log
timeout 900 python bench.py --no-prefill --no-cpu-baseline --no-parity-sample > $O/bench_dec_r02p.json 2>$O/bench_dec_r02p.err
echo "bench rc=$?"; python -c "
import json;d=json.loads(open('$O/bench_dec_r02p.json').read().strip().splitlines()[-1]);print(d['value'],d['dense_us_per_token'],d['gpu_launches'],d['e2e']['value'])
for c in d.get('configs',[]): print(json.dumps(c)[:300])"
