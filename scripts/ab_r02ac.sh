# A/B (same box): layer 0's selection on its own stream (working tree engine.py) vs HEAD's engine.py
set -u
O=gpurun_out; mkdir -p $O
E=paper_2512_16391_b200/engine.py
timeout 1200 python -m pytest tests/test_decode_gpu.py tests/test_scale_gpu.py -q -x -rf > $O/t_r02ac.log 2>&1
echo "tests rc=$?"; tail -2 $O/t_r02ac.log
cp $E /tmp/engine_new.py
for i in 1 2; do
  cp /tmp/engine_new.py $E
  timeout 600 python bench.py --no-prefill --no-cpu-baseline --no-configs --no-parity-sample > $O/bac_new_$i.json 2>/dev/null
  cp _exp/engine_head.py $E
  timeout 600 python bench.py --no-prefill --no-cpu-baseline --no-configs --no-parity-sample > $O/bac_head_$i.json 2>/dev/null
done
cp /tmp/engine_new.py $E
for f in $O/bac_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',d['value'],d['dense_us_per_token'],d['e2e']['value'])"; done
