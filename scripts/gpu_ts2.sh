cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --timestamps 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['config']['kernel_ms'])"
