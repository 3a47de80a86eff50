# GPU tests + C3 / C5 bench lines + one ncu --set full capture of a kernel ($KERNEL_MANGLED regex)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-v}
if [ -z "$SKIP_TESTS" ]; then
timeout 900 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/gpu_tests_$TAG.log
fi
for cfg in ${CONFIGS:-c3}; do
  extra=""; [ $cfg = c5 ] && extra="--warmup 2" || extra="--steps 10 --warmup 3"
  timeout 1500 python bench.py --config $cfg $extra $BENCH_EXTRA > gpurun_out/bench_${cfg}_$TAG.json 2> gpurun_out/bench_${cfg}_$TAG.err
  echo "$cfg rc=$?"; python - <<PY || tail -5 gpurun_out/bench_${cfg}_$TAG.err
import json; d=json.load(open('gpurun_out/bench_${cfg}_$TAG.json'))
print('$cfg ms', d['ms_per_step'], 'e2e', d['e2e'].get('ms_per_frame'), 'parity', {k: d.get('parity', {}).get(k) for k in ('pixel_mismatches', 'pass_stat_mismatches', 'renders_checked')} if d.get('parity') else None)
if 'stage_ms_per_frame' in d: print(' stages', d['stage_ms_per_frame'])
if 'kernels' in d:
    for k in d['kernels'][:10]: print('  ', k['kernel'][:60], k['ms_per_frame'], k['gbs'])
if 'frame_ms' in d: print(' c5 frame ms', d['frame_ms']['mean'], d['frame_ms']['median'], d['frame_ms']['max'])
PY
done
if [ -n "$KERNEL_MANGLED" ]; then
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:$KERNEL_MANGLED -s ${SKIP:-4} -c 1 \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo full_rc=$?
tail -3 gpurun_out/ncu_full_$TAG.log
fi
