set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in yelp clf; do timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --config $c > gpurun_out/bench_$c.log 2>&1; tail -1 gpurun_out/bench_$c.log; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_taxi.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --config taxi > gpurun_out/ncu_launch_taxi.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan -s 2 -c 1 -o gpurun_out/prof_taxi1g python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config taxi --records 10000000 > gpurun_out/ncu_full_taxi.log 2>&1; echo ncu2 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan -s 2 -c 1 -o gpurun_out/prof_yelp1g python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config yelp --records 1400000 > gpurun_out/ncu_full_yelp.log 2>&1; echo ncu3 rc=$?
ls -la gpurun_out
