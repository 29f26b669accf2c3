# A/B (same box): hoisted schedule (big kernels on the main stream, selections on the side) vs HEAD's overlap
set -u
O=gpurun_out; mkdir -p $O
E=paper_2512_16391_b200/engine.py
cp $E /tmp/engine_new.py
timeout 1200 python -m pytest tests/test_decode_gpu.py tests/test_scale_gpu.py -q -x -rf > $O/t_r02ag.log 2>&1
echo "tests rc=$?"; tail -1 $O/t_r02ag.log
python scripts/timeline_step.py > $O/timeline_hoist.txt 2>&1; cat $O/timeline_hoist.txt
for i in 1 2; do
  cp /tmp/engine_new.py $E
  timeout 600 python bench.py --no-prefill --no-cpu-baseline --no-parity-sample --no-configs > $O/bah_new_$i.json 2>/dev/null
  cp _exp/engine_head.py $E
  timeout 600 python bench.py --no-prefill --no-cpu-baseline --no-parity-sample --no-configs > $O/bah_head_$i.json 2>/dev/null
done
cp /tmp/engine_new.py $E
for f in $O/bah_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',d['value'],d['dense_us_per_token'],d['e2e']['value'])"; done
