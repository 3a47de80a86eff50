# GPU parity tests, then the C3 bench line and the C4 / C5 configuration lines
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_c3.json 2> gpurun_out/cfg_c3.err; echo c3_rc=$?
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_c4.json 2> gpurun_out/cfg_c4.err; echo c4_rc=$?
timeout 900 python bench.py --config c5 --warmup 3 > gpurun_out/cfg_c5.json 2> gpurun_out/cfg_c5.err; echo c5_rc=$?
tail -3 gpurun_out/cfg_c5.err
