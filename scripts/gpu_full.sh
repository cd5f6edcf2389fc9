cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 600 python -m pytest tests -m gpu -q -x --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_full.log
for c in yelp clf; do timeout 600 python bench.py --config $c --no-e2e --no-cpu > gpurun_out/bench_$c.log 2>&1; echo bench $c rc=$?; tail -1 gpurun_out/bench_$c.log; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_taxi.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_emit -s 3 -c 1 -o gpurun_out/prof_taxi_emit python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full_taxi.log 2>&1; echo ncu2 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 6 -c 2 -o gpurun_out/prof_taxi_pass python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full_taxi2.log 2>&1; echo ncu3 rc=$?
