# decode step: side-stream groups (and their main-stream launches) in reverse layer order vs HEAD
set -u
O=gpurun_out; mkdir -p $O
E=paper_2512_16391_b200/engine.py
cp $E /tmp/engine_cur.py
cp _exp/engine_rev.py $E; timeout 900 python -m pytest tests/test_decode_gpu.py -q -x -k "multi_layer or all_heads or llama" > $O/t_r02ap.log 2>&1; echo "tests rc=$?"; tail -1 $O/t_r02ap.log
for i in 1 2; do
  for v in head rev; do
    cp _exp/engine_$v.py $E
    timeout 600 python bench.py --no-prefill --no-cpu-baseline --no-parity-sample --no-configs --no-e2e > $O/bar_${v}_$i.json 2>/dev/null
  done
done
cp /tmp/engine_cur.py $E
for f in $O/bar_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',d['value'],d['dense_us_per_token'])"; done
