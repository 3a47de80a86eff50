# Round evidence: C3 bench line (+ CPU baseline), reference arm, C4/C5 lines, rank shares,
# the C2 speculation sweep, the ncu launch list and --set full captures.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/gpu_tests.log
timeout 1200 python bench.py > gpurun_out/ev_c3.json 2> gpurun_out/ev_c3.err; echo c3_rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev_ref.json 2> gpurun_out/ev_ref.err; echo ref_rc=$?
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev_c4.json 2> gpurun_out/ev_c4.err; echo c4_rc=$?
timeout 900 python bench.py --config c5 --warmup 3 > gpurun_out/ev_c5.json 2> gpurun_out/ev_c5.err; echo c5_rc=$?
for n in 2 4 8; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --rank-share $n > gpurun_out/ev_rs$n.json 2> gpurun_out/ev_rs$n.err; echo rs${n}_rc=$?
done
for m in 1 2 4 8 16 32 64; do
  timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline --max-spec $m > gpurun_out/ev_c2_s$m.json 2> gpurun_out/ev_c2_s$m.err; echo c2_s${m}_rc=$?
done
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 3000 --csv --log-file gpurun_out/ev_launches.csv $CMD > gpurun_out/ev_ncu_launches.log 2>&1; echo launches_rc=$?
for spec in "k_iso_cell_mask:1" "k_rt_shade:1" "k_bitmap_dense:2"; do
  k=${spec%%:*}; s=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 \
      -f -o gpurun_out/full_${k}_$s $CMD > gpurun_out/ncu_full_${k}.log 2>&1; echo "$k full_rc=$?"
done
