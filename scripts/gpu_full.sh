# one `ncu --set full` capture per kernel regex given (the same bench command first exits 0 without ncu)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline ${BENCH_ARGS}"
SKIP=${SKIP:-5}
timeout 600 $CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err || { echo plain_failed; exit 1; }
for K in "$@"; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 \
      -o gpurun_out/prof_$K -f $CMD > gpurun_out/ncu_full_$K.log 2>&1; echo full_${K}_rc=$?
done
