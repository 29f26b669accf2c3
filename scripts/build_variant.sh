#!/usr/bin/env bash
# Build an experiment variant of the library (dev tool):
#   bash scripts/build_variant.sh NAME -DKSCD_EXP=1 ...  ->  _exp/libkascade_NAME.so
set -e
NAME=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p $R/_exp/$NAME
for f in $R/paper_2512_16391_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
    -Xcompiler -fPIC,-O2 -I $R/paper_2512_16391_b200/csrc -I $R/include "$@" -c $f -o $R/_exp/$NAME/$(basename $f .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/_exp/libkascade_$NAME.so $R/_exp/$NAME/*.o -lcudart
rm -rf $R/_exp/$NAME
echo $R/_exp/libkascade_$NAME.so
