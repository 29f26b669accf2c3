# A/B (same box): side stream (score passes + selections) at high priority vs default
set -u
O=gpurun_out; mkdir -p $O
E=paper_2512_16391_b200/engine.py
cp $E /tmp/engine_cur.py
for i in 1 2; do
  for v in head mainhp; do
    cp _exp/engine_$v.py $E
    timeout 600 python bench.py --no-prefill --no-cpu-baseline --no-parity-sample --no-configs > $O/baf_${v}_$i.json 2>/dev/null
  done
done
cp /tmp/engine_cur.py $E
for f in $O/baf_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',d['value'],d['dense_us_per_token'],d['e2e']['value'],[ (c.get('kascade_us_per_token') or c.get('decode_kascade_us_per_token')) for c in d['configs']])"; done
