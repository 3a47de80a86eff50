# Final round evidence: tests, C3 bench line (+ CPU baseline), rank shares, ncu launch list.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/gpu_tests.log
timeout 1200 python bench.py > gpurun_out/ev_c3.json 2> gpurun_out/ev_c3.err; echo c3_rc=$?
for n in 2 4 8; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --rank-share $n > gpurun_out/ev_rs$n.json 2> gpurun_out/ev_rs$n.err; echo rs${n}_rc=$?
done
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev_c4.json 2> gpurun_out/ev_c4.err; echo c4_rc=$?
timeout 900 python bench.py --config c5 --warmup 3 > gpurun_out/ev_c5.json 2> gpurun_out/ev_c5.err; echo c5_rc=$?
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 3000 --csv --log-file gpurun_out/ev_launches.csv $CMD > gpurun_out/ev_ncu_launches.log 2>&1; echo launches_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rt_shade -s 1 -c 1 \
    -f -o gpurun_out/full_k_rt_shade_1 $CMD > gpurun_out/ncu_full_k_rt_shade.log 2>&1; echo "shade full_rc=$?"
