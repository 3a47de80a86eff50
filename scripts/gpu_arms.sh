# reference arm (CPU oracle port, all host threads) + B200 arm with cpu_baseline + forced NCCL shard path
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_arm.json 2> gpurun_out/ref_arm.err; echo ref_rc=$?
tail -c 1500 gpurun_out/ref_arm.json; tail -3 gpurun_out/ref_arm.err
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo b200_rc=$?
python scripts/show_bench.py gpurun_out/bench_c3.json; python -c "
import json; d=json.load(open('gpurun_out/bench_c3.json')); print('e2e', d['e2e']); print('roofline', d['roofline']); print('cpu', d.get('cpu_baseline')); print('parity', d.get('parity')); print('clocks', d['clocks'], 'launches', d['gpu_launches'])"
tail -3 gpurun_out/bench_c3.err
timeout 600 python bench.py --force-shard --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/shard1.json 2> gpurun_out/shard1.err; echo shard_rc=$?
python scripts/show_bench.py gpurun_out/shard1.json; tail -3 gpurun_out/shard1.err
