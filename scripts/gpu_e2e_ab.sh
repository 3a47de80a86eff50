# e2e A/B: render() end to end (WAVECAST_TRACE split) for the working tree and $VARIANTS
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_streaming.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/e2e_tests.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/e2e_tests.log)"
for v in default $VARIANTS; do
  if [ $v = default ]; then unset WAVECAST_LIB; else export WAVECAST_LIB=$PWD/paper_2309_10212_b200/variants/lib_$v.so; fi
  for cfg in ${CONFIGS:-c3}; do
    timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 ${BENCH_EXTRA:---no-cpu-baseline} > gpurun_out/e2e_${cfg}_$v.json 2> gpurun_out/e2e_${cfg}_$v.err
    python -c "
import json; d=json.load(open('gpurun_out/e2e_${cfg}_$v.json')); p=d.get('parity') or {}
print('$v', '$cfg', d['ms_per_step'], 'e2e', d['e2e']['ms_per_frame'], 'mism', p.get('pixel_mismatches'))"
  done
done
