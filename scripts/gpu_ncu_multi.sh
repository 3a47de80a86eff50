# --set full captures of several kernels of `bench.py --steps 1 --warmup 1` in one call.
# usage: bash scripts/gpu_ncu_multi.sh "regex1:skip1" "regex2:skip2" ...  (BENCH_ARGS optional)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline ${BENCH_ARGS}"
timeout 600 $CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err; echo plain_rc=$?
for spec in "$@"; do
  k=${spec%%:*}; s=${spec##*:}
  tag=$(echo "$k" | tr -c 'A-Za-z0-9_\n' '_')
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 \
      -f -o gpurun_out/full_${tag}_$s $CMD > gpurun_out/ncu_full_${tag}.log 2>&1; echo "$k full_rc=$?"
done
