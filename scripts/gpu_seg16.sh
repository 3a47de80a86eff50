# half-warp-per-ray traversal: parity with it forced on every thread-per-ray pass, then timing variants
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
WAVECAST_LIB=$PWD/paper_2309_10212_b200/variants/lib_s16all.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py -x -q -p no:cacheprovider > gpurun_out/t16.log 2>&1; echo "forced-16 tests: $(tail -1 gpurun_out/t16.log)"
VARIANTS="$VARIANTS" bash scripts/gpu_grid.sh
for v in default $VARIANTS; do
  if [ $v = default ]; then unset WAVECAST_LIB; else export WAVECAST_LIB=$PWD/paper_2309_10212_b200/variants/lib_$v.so; fi
  for n in 4 2; do
    timeout 600 python bench.py --rank-share $n --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$v share$n', d['ms_per_step'], d['pass_ms'])"
  done
done
