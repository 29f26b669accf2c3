# final validation of the committed code: all GPU tests and smoke()
set -u
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -rf > $O/tests_final.log 2>&1
echo "tests rc=$?"; tail -2 $O/tests_final.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_final.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke_final.log
