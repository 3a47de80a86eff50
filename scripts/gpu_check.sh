set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -3 gpurun_out/smoke.log
timeout 900 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
tail -15 gpurun_out/gpu_tests.log
