# reset-stage variants: C3 frame time and the reset stage's device ms
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in default $VARIANTS; do
  if [ $v = default ]; then unset WAVECAST_LIB; else export WAVECAST_LIB=$PWD/paper_2309_10212_b200/variants/lib_$v.so; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$v', d['ms_per_step'], 'reset', d['stage_ms_per_frame']['reset'], 'first', d.get('time_to_first_pass_ms'), 'passes', d['pass_ms'])"
done
