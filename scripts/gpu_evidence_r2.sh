# Round-2 evidence on the final code: bench lines for every BASELINE config
# (with full-frame oracle parity), the C2 speculation sweep, one rank's share
# of 2/4/8-way splits, the NCCL data plane on one GPU, the reference arm, and
# an ncu launch list of a C3 run.  Outputs -> gpurun_out/ev_*.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() { name=$1; shift; timeout 1500 python bench.py "$@" > gpurun_out/ev_$name.json 2> gpurun_out/ev_$name.err; echo "$name rc=$?"; }
run c3 --steps 20 --warmup 3 --dump-kernels
run c2 --config c2 --steps 10 --warmup 3
run c4 --config c4 --steps 10 --warmup 3
run c5 --config c5 --warmup 2
for m in 1 2 4 8 16 32 64; do run c2_ms$m --config c2 --max-spec $m --steps 10 --warmup 3 --no-cpu-baseline; done
for n in 2 4 8; do run share$n --rank-share $n --steps 10 --warmup 3 --no-cpu-baseline; done
run c3_spec1 --max-spec 1 --steps 3 --warmup 3
run shard1 --force-shard --steps 10 --warmup 3 --no-cpu-baseline
run reference --impl reference --steps 3 --warmup 1
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/ev_launch_plain.json 2> gpurun_out/ev_launch_plain.err && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 3000 --csv --log-file gpurun_out/ev_launches.csv $CMD > gpurun_out/ev_ncu_launches.log 2>&1; echo launches_rc=$?
