#!/usr/bin/env bash
# One GPU session: tests, the bench line, the bench's ncu launch list and
# --set full captures of the two roofline kernels at bench shapes.
#   gpurun --timeout 3000 -- 'bash scripts/gpu_round.sh TAG [tests|bench|ncu ...]'
set -u
TAG=${1:-r01}
shift || true
STEPS=${*:-tests bench launches full}
O=gpurun_out
mkdir -p $O
for s in $STEPS; do
  case $s in
    tests)
      timeout 1500 python -m pytest tests -m gpu -x -q > $O/tests_$TAG.log 2>&1
      echo "tests rc=$?"; tail -3 $O/tests_$TAG.log ;;
    bench)
      timeout 1200 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err
      echo "bench rc=$?"; tail -c 600 $O/bench_$TAG.json ;;
    launches)
      timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file $O/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-configs \
        > $O/launches_$TAG.out 2>&1
      echo "launches rc=$?" ;;
    full)
      timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
        -k 'regex:decode_attn_kernel<\(int\)1' -s 2 -c 1 -o $O/full_sparse_decode_$TAG -f \
        python scripts/prof_kernels.py decode > $O/full_dec_$TAG.out 2>&1
      echo "full decode rc=$?"
      timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
        -k 'regex:prefill_attn_kernel<\(int\)1' -s 1 -c 1 -o $O/full_sparse_prefill_$TAG -f \
        python scripts/prof_kernels.py prefill 131072 > $O/full_pre_$TAG.out 2>&1
      echo "full prefill rc=$?" ;;
  esac
done
