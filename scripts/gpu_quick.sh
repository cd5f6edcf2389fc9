# usage (GPU box): bash scripts/gpu_quick.sh <tag> : GPU tests + yelp/taxi/clf bench lines (fused and staged)
cd $GRAFT_REPO_ROOT
tag=$1; O=gpurun_out/$tag; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
for c in ${CONFIGS:-yelp taxi clf}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu > $O/bench_$c.log 2>&1; echo "bench $c rc=$?"; tail -1 $O/bench_$c.log | cut -c1-200
  python -c "import json,sys; l=json.loads(open('$O/bench_$c.log').read().strip().splitlines()[-1]); print(l['value'], l['config']['kernel_ms'], l['roofline']['step_frac'] if l.get('roofline') else None)" 2>/dev/null
  if [ -n "$STAGED" ]; then PARPA_STAGED=1 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu > $O/bench_${c}_staged.log 2>&1; echo "staged $c rc=$?";
  python -c "import json,sys; l=json.loads(open('$O/bench_${c}_staged.log').read().strip().splitlines()[-1]); print(l['value'], l['config']['kernel_ms'])" 2>/dev/null; fi
done
