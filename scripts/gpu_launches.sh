# ncu launch list (time + DRAM bytes per kernel) of `bench.py --steps 1 --warmup 1`, after the same command exits 0.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline ${BENCH_ARGS}"
timeout 600 $CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none ${NCU_EXTRA} \
    -c 3000 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo launches_rc=$?
