# GPU parity tests against an alternative library build ($1 = path)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
WAVECAST_LIB=$PWD/$1 timeout 900 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_var.log 2>&1; echo "tests[$1]_rc=$?"; tail -2 gpurun_out/gpu_tests_var.log
