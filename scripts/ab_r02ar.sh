# decode score writes as streaming stores (st.global.cs) vs default
set -u
O=gpurun_out; mkdir -p $O
for i in 1 2; do
  echo "== default"; python scripts/perf_decode_ops.py 8 32 8 131072 2>&1 | grep -E "dense_scores|scores_pass1"
  echo "== stcs"; KSCD_LIB_PATH=$PWD/_exp/libkascade_stcs.so python scripts/perf_decode_ops.py 8 32 8 131072 2>&1 | grep -E "dense_scores|scores_pass1"
done
for i in 1 2; do
  timeout 600 python bench.py --no-prefill --no-cpu-baseline --no-parity-sample --no-configs --no-e2e > $O/bas_def_$i.json 2>/dev/null
  KSCD_LIB_PATH=$PWD/_exp/libkascade_stcs.so timeout 600 python bench.py --no-prefill --no-cpu-baseline --no-parity-sample --no-configs --no-e2e > $O/bas_stcs_$i.json 2>/dev/null
done
for f in $O/bas_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',d['value'],d['dense_us_per_token'])"; done
