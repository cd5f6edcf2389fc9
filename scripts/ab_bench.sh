# usage (GPU box): bash scripts/ab_bench.sh "<configs>" : bench lines (value + kernel ms) per ab/libparpa_*.so
cd $GRAFT_REPO_ROOT
for c in $1; do for f in ab/libparpa_*.so; do
  echo "== $c $f"
  PARPA_LIB=$PWD/$f timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu --parity ${PARITY:-none} 2>&1 | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    j=json.loads(l); print(j['value'], j['config']['kernel_ms'], 'parity', (j.get('parity') or {}).get('ok'))"
done; done
