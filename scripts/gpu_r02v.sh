# final evidence after the pass-B tail change: GPU tests, smoke, bench line, launch list
set -u
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -rf > $O/tests_r02v.log 2>&1
echo "tests rc=$?"; tail -1 $O/tests_r02v.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_r02v.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke_r02v.log
bash scripts/gpu_r02.sh r02v bench launches
