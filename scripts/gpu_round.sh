# tests + smoke + C3 bench (+ optional ncu full capture of one kernel)
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
tail -5 gpurun_out/gpu_tests.log
timeout 1200 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3_rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_c3.json'))
print('ms/frame', d['ms_per_step'], 'Mrays/s', d['value'], 'e2e', d['e2e']['value'], 'stages', d['stage_ms_per_frame'])
print('roofline', d['roofline']); print('cpu', d.get('cpu_baseline')); print('parity', d.get('parity')); print('clocks', d['clocks'])"
tail -3 gpurun_out/bench_c3.err
if [ -n "$1" ]; then
  CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
  timeout 600 $CMD > gpurun_out/prof_plain.json 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$1 -s ${2:-5} -c 1 \
      -o gpurun_out/prof_$1 $CMD > gpurun_out/ncu_full.log 2>&1; echo full_rc=$?
  tail -2 gpurun_out/ncu_full.log
fi
