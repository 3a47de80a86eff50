# The GPU parity suite against the checked build (-DWC_CHECKS=1: device-side
# index checks that trap), standing in for compute-sanitizer memcheck, which is
# closed on this pool.  Log -> gpurun_out/checked_tests.log
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
WAVECAST_LIB=$PWD/paper_2309_10212_b200/variants/lib_checked.so timeout 1500 \
  python -m pytest tests/ -m gpu -q -p no:cacheprovider > gpurun_out/checked_tests.log 2>&1
echo "checked_rc=$?"; tail -3 gpurun_out/checked_tests.log
