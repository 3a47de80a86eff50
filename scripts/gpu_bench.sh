set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3_rc=$?
tail -c 5000 gpurun_out/bench_c3.json; tail -5 gpurun_out/bench_c3.err
