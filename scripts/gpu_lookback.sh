# CTA-wide look-back vs the warp form (variants), C3 + C2 at max_spec 1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_lb.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/gpu_tests_lb.log
for v in default lbwarp lbk1 lbk2; do
  if [ $v = default ]; then unset WAVECAST_LIB; else export WAVECAST_LIB=$PWD/paper_2309_10212_b200/variants/lib_$v.so; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/lb_c3_$v.json 2> gpurun_out/lb_c3_$v.err
  timeout 600 python bench.py --config c2 --max-spec 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/lb_c2s1_$v.json 2> gpurun_out/lb_c2s1_$v.err
  python - <<PY
import json
for c in ('c3','c2s1'):
    try:
        d=json.load(open('gpurun_out/lb_%s_$v.json'%c))
        print('$v', c, d['ms_per_step'], 'pass_ms', d.get('pass_ms')[:6], 'mark', d['stage_ms_per_frame'].get('mark'))
    except Exception as e: print('$v', c, 'ERR', e)
PY
done
