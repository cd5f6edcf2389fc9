cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 600 python -m pytest tests -m gpu -q -x --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
export PARPA_DEBUG=1
for w in yelp taxi; do timeout 120 python scripts/probe.py $w 1e9 fused 2>&1 | grep -E "per-CTA|ok|MISMATCH|Error" | tail -3; done
unset PARPA_DEBUG
for c in yelp taxi clf; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --config $c > gpurun_out/bench_$c.log 2>&1; echo bench $c rc=$?; tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], 'GB/s', d['ms_per_step'], 'ms', 'frac', d['roofline']['frac'], d['config']['kernel_ms'])" 2>&1 | tail -1
done
