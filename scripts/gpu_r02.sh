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
