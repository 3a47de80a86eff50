# one ncu --set full capture of kernel $1 (skip $2 launches) of a short bench run
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline ${BENCH_ARGS}"
timeout 600 $CMD > gpurun_out/prof_plain.json 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$1 -s ${2:-5} -c 1 \
    -o gpurun_out/prof_$1 $CMD > gpurun_out/ncu_full.log 2>&1; echo full_rc=$?
tail -2 gpurun_out/ncu_full.log
