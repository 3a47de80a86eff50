# bench the default build and each variant in $VARIANTS over the argument sets in
# $ARGSETS (";"-separated bench.py argument lists); optional parity subset per variant
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
IFS=';' read -ra SETS <<< "${ARGSETS:---config c3}"
for v in default $VARIANTS; do
  if [ $v = default ]; then unset WAVECAST_LIB; else export WAVECAST_LIB=$PWD/paper_2309_10212_b200/variants/lib_$v.so; fi
  if [ -n "$PARITY" ]; then
    timeout 900 python -m pytest $PARITY -x -q -p no:cacheprovider > gpurun_out/var_parity_$v.log 2>&1; echo "$v parity rc=$? $(tail -1 gpurun_out/var_parity_$v.log)"
  fi
  k=0
  for args in "${SETS[@]}"; do
    k=$((k+1))
    timeout 900 python bench.py $args --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/var_${k}_$v.json 2> gpurun_out/var_${k}_$v.err
    python - <<PY
import json
try:
    d=json.load(open('gpurun_out/var_${k}_$v.json'))
    ks={k['kernel'][:20]: k['ms_per_frame'] for k in d['kernels'][:6]}
    print('$v', '[$args]', d['ms_per_step'], 'pass_ms', d.get('pass_ms')[:5], ks)
except Exception as e: print('$v', '[$args]', 'ERR', e)
PY
  done
done
