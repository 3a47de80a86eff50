cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for lib in paper_2309_10212_b200/variants/lib_*.so; do
  name=$(basename $lib .so)
  for r in 1 8; do
    WAVECAST_LIB=$PWD/$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --rank-share $r > gpurun_out/v_${name}_$r.json 2>/dev/null
    python scripts/show_bench.py gpurun_out/v_${name}_$r.json | head -1
  done
done
