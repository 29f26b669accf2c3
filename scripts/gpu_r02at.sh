set -u
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/tests_r02at.log 2>&1
echo "tests rc=$?"; tail -1 $O/tests_r02at.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash scripts/gpu_r02.sh r02at sanitize
KSCD_LIB_PATH=$PWD/_exp/libkascade_pbtrace.so python scripts/pb_trace.py 131072 2>&1 | tail -1
for i in 1 2; do timeout 300 python scripts/perf_prefill.py 131072; done
