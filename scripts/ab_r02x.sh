# decode select launched programmatically (pool / Top-k PDL): tests + decode bench, and the HEAD lib for A/B
set -u
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_decode_gpu.py tests/test_scale_gpu.py tests/test_prefill_gpu.py tests/test_pre_pooling_gpu.py -q -x -rf > $O/t_r02x.log 2>&1
echo "tests rc=$?"; tail -2 $O/t_r02x.log
for i in 1 2; do
  KSCD_LIB_PATH=$PWD/_exp/libkascade_base2.so timeout 600 python bench.py --no-prefill --no-cpu-baseline --no-configs --no-parity-sample --no-e2e > $O/bx_base_$i.json 2>/dev/null
  timeout 600 python bench.py --no-prefill --no-cpu-baseline --no-configs --no-parity-sample --no-e2e > $O/bx_new_$i.json 2>/dev/null
done
for f in $O/bx_*.json; do python -c "
import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',d['value'],d['dense_us_per_token'],d['ms_per_step'])"; done
