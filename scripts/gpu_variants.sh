# bench C3 (+ optional C4) for the default build and each variant in $VARIANTS
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
if [ -z "$SKIP_TESTS" ]; then
timeout 900 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_var.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/gpu_tests_var.log
fi
for v in default $VARIANTS; do
  if [ $v = default ]; then unset WAVECAST_LIB; else export WAVECAST_LIB=$PWD/paper_2309_10212_b200/variants/lib_$v.so; fi
  for cfg in ${CONFIGS:-c3}; do
    timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline $BENCH_EXTRA > gpurun_out/var_${cfg}_$v.json 2> gpurun_out/var_${cfg}_$v.err
    python - <<PY
import json
try:
    d=json.load(open('gpurun_out/var_${cfg}_$v.json'))
    ks={k['kernel'][:28]: k['ms_per_frame'] for k in d['kernels'][:8]}
    print('$v', '$cfg', d['ms_per_step'], 'e2e', d['e2e'].get('ms_per_frame'), 'pass_ms', d.get('pass_ms')[:5], ks)
except Exception as e: print('$v', '$cfg', 'ERR', e)
PY
  done
done
