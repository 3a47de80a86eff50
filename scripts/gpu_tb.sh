# parity tests, then C3 bench lines (args per line of $VARIANTS, default: plain C3 and --rank-share 8)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -15 gpurun_out/gpu_tests.log | grep -E "passed|failed|Error|assert" | head -8
i=0
while IFS= read -r args; do
  i=$((i+1))
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $args > gpurun_out/q_$i.json 2> gpurun_out/q_$i.err
  echo "variant $i: [$args]"; python scripts/show_bench.py gpurun_out/q_$i.json || tail -3 gpurun_out/q_$i.err
done <<< "${VARIANTS:-
--rank-share 8}"
