# Round-2 evidence refresh on the final code (same legs as gpu_evidence_r2.sh)
# + the GPU test suite log + ncu --set full captures of the top kernels.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -q -p no:cacheprovider > gpurun_out/ev_gpu_tests.log 2>&1; echo tests_rc=$?
bash scripts/gpu_evidence_r2.sh
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
for k in '^k_traverse$' k_rt_find k_decode_insert k_mark_extract; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 \
      -o gpurun_out/ev_full_$(echo $k | tr -d "^$") $CMD > gpurun_out/ev_full_$(echo $k | tr -d "^$").log 2>&1; echo "full $k rc=$?"
done
