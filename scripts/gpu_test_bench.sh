# usage: bash scripts/gpu_test_bench.sh [configs...]   (runs on the GPU box)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/pytest_gpu.log
for c in ${@:-taxi yelp clf}; do
  timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --config $c > gpurun_out/bench_$c.log 2>&1; echo bench $c rc=$?; tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], 'GB/s', d['ms_per_step'], 'ms', 'frac', d['roofline']['frac'], d['config']['kernel_ms'])" 2>&1 | tail -1
done
