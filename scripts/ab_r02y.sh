# decode step vs the tcgen05 dense / score pass's CTA waves per layer (KSCD_DTC_WAVES)
set -u
O=gpurun_out; mkdir -p $O
for i in 1 2; do
  for v in w6 w8 w12 w16 w24; do
    KSCD_LIB_PATH=$PWD/_exp/libkascade_$v.so timeout 600 python bench.py --no-prefill --no-cpu-baseline --no-configs --no-parity-sample --no-e2e > $O/bz_${v}_$i.json 2>/dev/null
  done
  timeout 600 python bench.py --no-prefill --no-cpu-baseline --no-configs --no-parity-sample --no-e2e > $O/bz_w4_$i.json 2>/dev/null
done
for f in $O/bz_*.json; do python -c "
import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',d['value'],d['dense_us_per_token'],d['per_layer_ms'])"; done
