cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 600 python -m pytest tests -m gpu -q -x --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
for c in yelp taxi clf; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --config $c > gpurun_out/bench_$c.log 2>&1; echo bench $c rc=$?; tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], 'GB/s', d['ms_per_step'], 'ms', 'frac', d['roofline']['frac'], d['config']['kernel_ms'])" 2>&1 | tail -1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_scan -s 2 -c 1 -o gpurun_out/prof_taxi_v3 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config taxi --records 10000000 > gpurun_out/ncu_taxi_v3.log 2>&1; echo ncu rc=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_scan -s 2 -c 1 -o gpurun_out/prof_yelp_v3 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config yelp --records 1400000 > gpurun_out/ncu_yelp_v3.log 2>&1; echo ncu rc=$?
