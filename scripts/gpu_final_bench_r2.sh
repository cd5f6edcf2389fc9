# Round-2 final evidence, part 2 (one B200): smoke, GPU tests, the default bench line (yelp + taxi / clf / cfg1
# sub-records with full parity), the reference arm, taxi64 and the rate-vs-size sweep.
cd $GRAFT_REPO_ROOT
O=gpurun_out/final; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -1 $O/smoke.log
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > $O/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 $O/pytest_gpu.log
timeout 1500 python bench.py > $O/bench_default.log 2> $O/bench_default.err; echo bench rc=$?
timeout 900 python bench.py --impl reference > $O/bench_reference.log 2>&1; echo ref rc=$?
timeout 1200 python bench.py --config taxi64 --steps 3 --warmup 1 > $O/bench_taxi64.log 2> $O/bench_taxi64.err; echo taxi64 rc=$?
timeout 900 python scripts/size_sweep.py yelp taxi > $O/size_sweep.jsonl 2> $O/size_sweep.err; echo sweep rc=$?
