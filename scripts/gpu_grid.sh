# grid-size variants: one rank's 8-way share, the whole C3 frame, C2 at max_spec 1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in default $VARIANTS; do
  if [ $v = default ]; then unset WAVECAST_LIB; else export WAVECAST_LIB=$PWD/paper_2309_10212_b200/variants/lib_$v.so; fi
  a=$(timeout 600 python bench.py --rank-share 8 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'], d['pass_ms'])")
  b=$(timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'], d['pass_ms'])")
  c=$(timeout 600 python bench.py --config c2 --max-spec 1 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'])")
  echo "$v | share8 $a | c3 $b | c2s1 $c"
done
