# ncu evidence for the bench: launch list with time + DRAM traffic for every kernel of
# `bench.py --steps 1 --warmup 1` (4 frames), and one --set full capture of kernel $1.
# Each ncu command runs only after the same command line exited 0 without ncu.
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
KERNEL=${1:-k_rt_solve}
SKIP=${2:-5}
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 3000 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo launches_rc=$?
timeout 600 $CMD > gpurun_out/prof_plain2.json 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$KERNEL -s $SKIP -c 1 \
    -o gpurun_out/prof_$KERNEL $CMD > gpurun_out/ncu_full.log 2>&1; echo full_rc=$?
tail -3 gpurun_out/ncu_full.log
