#!/usr/bin/env bash
# Round-2 GPU session helper:  bash scripts/gpu_r02.sh TAG step...
#   tests | sanitize | bench | launches | ncu_sparse_prefill | ncu_decode
set -u
TAG=${1:-r02}
shift || true
O=gpurun_out
mkdir -p $O
for s in "$@"; do
  case $s in
    tests)
      timeout 1800 python -m pytest tests -m gpu -q -s -rf --durations=10 > $O/tests_$TAG.log 2>&1
      echo "tests rc=$?"; tail -3 $O/tests_$TAG.log ;;
    sanitize)
      for tool in memcheck racecheck synccheck initcheck; do
        timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_cases.py \
          > $O/sanitizer_${tool}_$TAG.log 2>&1
        echo "$tool rc=$?"; tail -2 $O/sanitizer_${tool}_$TAG.log
      done ;;
    bench)
      timeout 1500 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err
      echo "bench rc=$?"; tail -c 400 $O/bench_$TAG.json; tail -3 $O/bench_$TAG.err ;;
    launches)
      timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file $O/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-configs \
        --no-parity-sample > $O/launches_$TAG.out 2>&1
      echo "launches rc=$?" ;;
  esac
done
# (appended) profiling steps: PROF=1 bash scripts/gpu_r02.sh TAG topk_ncu shard_ncu
for s in "$@"; do
  case $s in
    topk_ncu)
      timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
        -k 'regex:topk_kernel' -s 1 -c 1 -o $O/topk_$TAG -f python scripts/prof_kernels.py decode > $O/topk_ncu_$TAG.out 2>&1
      echo "topk ncu rc=$?" ;;
    shard_ncu)
      timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
        -k 'regex:decode_attn_kernel<\(int\)1' -s 1 -c 1 -o $O/shard_sparse_$TAG -f python scripts/prof_kernels.py decode_shard \
        > $O/shard_ncu_$TAG.out 2>&1
      echo "shard ncu rc=$?"
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/shard_launches_$TAG.csv \
        python scripts/prof_kernels.py decode_shard > /dev/null 2>&1
      echo "shard launches rc=$?" ;;
  esac
done
for s in "$@"; do
  case $s in
    newtests)
      timeout 1500 python -m pytest tests/test_pre_pooling_gpu.py tests/test_exporter_traces_gpu.py tests/test_decode_gpu.py \
        tests/test_compat_gpu.py tests/test_acceptance_gpu.py tests/test_shapes_gpu.py -q -s -rf > $O/newtests_$TAG.log 2>&1
      echo "newtests rc=$?"; grep -E "passed|failed|Error|swaps|rel-L2 engine" $O/newtests_$TAG.log | tail -30 ;;
    configs)
      timeout 1500 python bench.py --no-prefill --no-cpu-baseline --no-parity-sample > $O/configs_$TAG.json 2> $O/configs_$TAG.err
      echo "configs rc=$?"; tail -c 1500 $O/configs_$TAG.json ;;
  esac
done
for s in "$@"; do
  case $s in
    fullcap)
      timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
        -k 'regex:decode_attn_kernel' -s 3 -c 1 -o $O/step_reuse_run_$TAG -f python scripts/prof_step.py \
        > $O/fullcap_step_$TAG.out 2>&1
      echo "step reuse-run capture rc=$?"
      timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
        -k 'regex:pool_prefill' -s 1 -c 1 -o $O/pool_prefill_fused_$TAG -f python scripts/prof_kernels.py prefill 32768 \
        > $O/fullcap_pool_$TAG.out 2>&1
      echo "fused pass-B capture rc=$?"
      timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
        -k 'regex:prefill_attn_kernel<\(int\)1' -s 1 -c 1 -o $O/sparse_prefill_$TAG -f python scripts/prof_kernels.py prefill 131072 \
        > $O/fullcap_sp_$TAG.out 2>&1
      echo "sparse prefill capture rc=$?" ;;
  esac
done
