# bench each variant library (WAVECAST_LIB) on the C3 frame
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for lib in paper_2309_10212_b200/variants/lib_*.so; do
  name=$(basename $lib .so)
  WAVECAST_LIB=$PWD/$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/var_$name.json 2>gpurun_out/var_$name.err
  python -c "
import json,sys; d=json.load(open('gpurun_out/var_$name.json'))
print('$name', 'ms/frame', d['ms_per_step'], 'stages', d['stage_ms_per_frame'])" || tail -3 gpurun_out/var_$name.err
done
