# Checked build (-DWC_CHECKS=1) on the current code: GPU suite + C2/C3/C4
# full-frame parity; then an ncu --set full capture of k_traverse pass 0.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash scripts/gpu_checked.sh
for c in c2 c3 c4; do
  WAVECAST_LIB=$PWD/paper_2309_10212_b200/variants/lib_checked.so timeout 1200 python bench.py --config $c --steps 3 --warmup 3 \
     > gpurun_out/checked_$c.json 2> gpurun_out/checked_$c.err; echo "$c rc=$?"
done
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_traverse<' -s 0 -c 1 \
    -o gpurun_out/ev_full_trav_p0 $CMD > gpurun_out/ev_full_trav_p0.log 2>&1; echo "full trav p0 rc=$?"
