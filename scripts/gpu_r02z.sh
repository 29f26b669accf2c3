set -u
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x -rf > $O/tests_r02z.log 2>&1
echo "tests rc=$?"; tail -2 $O/tests_r02z.log
for i in 1 2; do
  KSCD_LIB_PATH=$PWD/_exp/libkascade_base2.so timeout 600 python bench.py --no-prefill --no-cpu-baseline --no-configs --no-parity-sample --no-e2e > $O/bzz_w4_$i.json 2>/dev/null
  timeout 600 python bench.py --no-prefill --no-cpu-baseline --no-configs --no-parity-sample --no-e2e > $O/bzz_new_$i.json 2>/dev/null
done
for f in $O/bzz_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',d['value'],d['dense_us_per_token'])"; done
