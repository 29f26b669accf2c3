set -u
O=gpurun_out; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:decode_attn_kernel' -s 3 -c 1 -o $O/step_reuse_run_r02n -f python scripts/prof_step.py > $O/fullcap_step_r02n.out 2>&1
echo "step capture rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:decode_tc_kernel' -s 1 -c 1 -o $O/step_score_r02n -f python scripts/prof_step.py > $O/fullcap_score_r02n.out 2>&1
echo "score capture rc=$?"
bash scripts/gpu_r02.sh r02n sanitize
