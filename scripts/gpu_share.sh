# one rank's share of an N-way tile split (bench --rank-share N) per variant, per-pass kernel rows
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in default $VARIANTS; do
  if [ $v = default ]; then unset WAVECAST_LIB; else export WAVECAST_LIB=$PWD/paper_2309_10212_b200/variants/lib_$v.so; fi
  for n in ${SHARES:-8}; do
    timeout 600 python bench.py --rank-share $n --steps 10 --warmup 3 --no-cpu-baseline --dump-kernels > gpurun_out/share${n}_$v.json 2> gpurun_out/share${n}_$v.err
    python - <<PY
import json
d=json.load(open('gpurun_out/share${n}_$v.json'))
rows=d.get('kernel_profile_rows') or []
trav=[(r['pass'], round(r['ms'],4)) for r in rows if r['kernel'].startswith('k_traverse')]
print('$v', 'N=$n', d['ms_per_step'], 'pass_ms', d.get('pass_ms'), 'trav', trav)
PY
  done
done
