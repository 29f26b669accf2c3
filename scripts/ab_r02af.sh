# A/B (same box): tcgen05 decode slot counts (dense K / V slots, score-pass K slots): 3/3/6 (current) vs smaller
# footprints that let the selection kernels co-reside on the SMs
set -u
O=gpurun_out; mkdir -p $O
for i in 1 2; do
  for v in s224 s223 s335; do
    KSCD_LIB_PATH=$PWD/_exp/libkascade_$v.so timeout 600 python bench.py --no-prefill --no-cpu-baseline --no-parity-sample --no-configs > $O/bag_${v}_$i.json 2>/dev/null
  done
  timeout 600 python bench.py --no-prefill --no-cpu-baseline --no-parity-sample --no-configs > $O/bag_cur_$i.json 2>/dev/null
done
for f in $O/bag_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',d['value'],d['dense_us_per_token'],d['e2e']['value'])"; done
KSCD_LIB_PATH=$PWD/_exp/libkascade_s224.so python scripts/timeline_step.py > $O/timeline_s224.txt 2>&1; cat $O/timeline_s224.txt
