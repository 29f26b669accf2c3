set -u
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x -rf > $O/tests_r02ab.log 2>&1
echo "tests rc=$?"; tail -2 $O/tests_r02ab.log
for i in 1 2; do
  timeout 600 python bench.py --no-prefill --no-cpu-baseline --no-configs --no-parity-sample > $O/bab_$i.json 2>$O/bab_$i.err
done
for f in $O/bab_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',d['value'],d['dense_us_per_token'],d['e2e']['value'],d['gpu_launches'])"; done
