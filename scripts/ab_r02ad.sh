# A/B (same box): HEAD engine vs split side streams (score passes | selections) vs split + layer 0's selection stream
set -u
O=gpurun_out; mkdir -p $O
E=paper_2512_16391_b200/engine.py
cp $E /tmp/engine_split.py
timeout 1200 python -m pytest tests/test_decode_gpu.py -q -x -rf > $O/t_r02ad.log 2>&1
echo "tests rc=$?"; tail -1 $O/t_r02ad.log
cp _exp/engine_sel0.py $E; timeout 1200 python -m pytest tests/test_decode_gpu.py -q -x -rf -k "multi_layer or host_step" > $O/t_r02ad_sel0.log 2>&1
echo "sel0 tests rc=$?"; tail -1 $O/t_r02ad_sel0.log
cp /dev/null /tmp/x
cp $E /tmp/engine_sel0.py
git_head=_exp/engine_head.py
for i in 1 2; do
  for v in head split; do
    case $v in head) cp _exp/engine_head.py $E;; split) cp /tmp/engine_split.py $E;; sel0) cp _exp/engine_sel0.py $E;; esac
    timeout 600 python bench.py --no-prefill --no-cpu-baseline --no-configs --no-parity-sample > $O/bad_${v}_$i.json 2>/dev/null
  done
done
cp /tmp/engine_split.py $E
for f in $O/bad_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',d['value'],d['dense_us_per_token'],d['e2e']['value'])"; done
