set -u
O=gpurun_out; mkdir -p $O
bash scripts/gpu_r02.sh r02au sanitize
timeout 900 python -m pytest tests/test_prefill_gpu.py tests/test_scale_gpu.py tests/test_pre_pooling_gpu.py -q -rf -k "prefill" 2>&1 | tail -1
for i in 1 2; do timeout 300 python scripts/perf_prefill.py 131072; done
