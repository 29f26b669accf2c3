# final round-2 evidence: GPU tests, smoke, bench line, launch list, prefill captures, per-block traces
set -u
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -rf > $O/tests_r02o.log 2>&1
echo "tests rc=$?"; tail -2 $O/tests_r02o.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_r02o.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke_r02o.log
bash scripts/gpu_r02.sh r02o bench launches
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:prefill_attn_kernel<\(int\)1' -s 1 -c 1 -o $O/sparse_prefill_r02o -f python scripts/prof_kernels.py prefill 131072 > $O/fullcap_sp_r02o.out 2>&1
echo "sparse prefill capture rc=$?"
KSCD_LIB_PATH=$PWD/_exp/libkascade_pftrace.so python scripts/pf_trace.py dense 32768 > $O/pf_trace_dense_32k_r02o.txt 2>&1
KSCD_LIB_PATH=$PWD/_exp/libkascade_pftrace.so python scripts/pf_trace.py sparse 131072 > $O/pf_trace_sparse_128k_r02o.txt 2>&1
head -6 $O/pf_trace_*_r02o.txt
