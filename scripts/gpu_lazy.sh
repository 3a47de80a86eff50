# lazy vs eager fine masks (WAVECAST_EAGER_MASKS=1): C3 frame / reset, 8-way share, C2 at max_spec 1, C4
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for mode in lazy eager; do
  if [ $mode = eager ]; then export WAVECAST_EAGER_MASKS=1; else unset WAVECAST_EAGER_MASKS; fi
  a=$(timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'], 'reset', d['stage_ms_per_frame']['reset'], d['pass_ms'], 'trav', d['stage_ms_per_frame']['traverse'])")
  b=$(timeout 600 python bench.py --rank-share 8 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'])")
  c=$(timeout 600 python bench.py --config c2 --max-spec 1 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'])")
  e=$(timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'])")
  echo "$mode | c3 $a | share8 $b | c2s1 $c | c4 $e"
done
