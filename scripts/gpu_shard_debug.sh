cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
NCCL_DEBUG=WARN timeout 600 python -X faulthandler -u bench.py --force-shard --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/shard1.log 2>&1; echo rc=$?
tail -30 gpurun_out/shard1.log
