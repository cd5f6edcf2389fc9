cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -q -x --timeout 200 2>&1 | tail -1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --timestamps 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ts', d['value'], d['config']['kernel_ms'])"
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('plain', d['value'], d['config']['kernel_ms'])"
