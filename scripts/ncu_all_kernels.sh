#!/usr/bin/env bash
# ncu --set full of every engine kernel at the bench shapes (one launch of
# each), for profiles/ncu_<tag>_kernels.md.
#   gpurun -- 'bash scripts/ncu_all_kernels.sh TAG'
TAG=${1:-r01}
O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:decode_attn|pool_decode|topk' -c 12 -o $O/all_decode_$TAG -f \
  python scripts/prof_kernels.py decode > $O/all_decode_$TAG.out 2>&1
echo "decode rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:prefill_attn|pool_prefill|topk' -c 5 -o $O/all_prefill_$TAG -f \
  python scripts/prof_kernels.py prefill 131072 > $O/all_prefill_$TAG.out 2>&1
echo "prefill rc=$?"
