# bench lines with full-frame oracle parity for every BASELINE config (C2-C5)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for cfg in c3 c2 c4; do
  timeout 900 python bench.py --config $cfg --steps ${STEPS:-5} --warmup 3 > gpurun_out/par_$cfg.json 2> gpurun_out/par_$cfg.err
  echo "$cfg rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/par_$cfg.json'))
print('$cfg', d['ms_per_step'], 'e2e', d['e2e']['ms_per_frame'], 'parity', d.get('parity'), 'roofline', d['roofline']['kernel'], d['roofline']['frac'])" || tail -5 gpurun_out/par_$cfg.err
done
timeout 1500 python bench.py --config c5 --warmup 2 > gpurun_out/par_c5.json 2> gpurun_out/par_c5.err
echo "c5 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/par_c5.json'))
print('c5', d['ms_per_step'], 'parity', d.get('parity'))" || tail -5 gpurun_out/par_c5.err
