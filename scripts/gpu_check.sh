set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
free -g | head -2; nproc
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -5 gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
tail -40 gpurun_out/gpu_tests.log
