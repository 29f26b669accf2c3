# sharded decode step: reuse runs as multi-layer launches (working tree) vs per-layer launches (HEAD)
set -u
S=paper_2512_16391_b200/sharding.py
cp $S /tmp/sharding_new.py
for i in 1 2; do
  cp /tmp/sharding_new.py $S; echo -n "multi: "; timeout 600 python scripts/perf_sharded_decode.py 2>&1 | tail -1
  cp _exp/sharding_head.py $S; echo -n "per-layer: "; timeout 600 python scripts/perf_sharded_decode.py 2>&1 | tail -1
done
cp /tmp/sharding_new.py $S
