# Round evidence on one B200 (run under gpurun): smoke, GPU tests, default bench (taxi with e2e and
# cpu_baseline), the reference arm, yelp / clf / cfg1 bench lines, the ncu launch list of the default
# bench command and one ncu --set full capture of k_emit / k_pass1 / k_pass2 per workload.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/ev
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -1 $O/smoke.log
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > $O/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 $O/pytest_gpu.log
timeout 1200 python bench.py > $O/bench_default.log 2>&1; echo bench rc=$?; tail -1 $O/bench_default.log | cut -c1-400
timeout 900 python bench.py --impl reference > $O/bench_reference.log 2>&1; echo ref rc=$?; tail -1 $O/bench_reference.log | cut -c1-300
for c in yelp clf cfg1; do timeout 900 python bench.py --config $c > $O/bench_$c.log 2>&1; echo bench $c rc=$?; tail -1 $O/bench_$c.log | cut -c1-300; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_taxi.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu_launch.log 2>&1; echo ncu-launch rc=$?
for c in taxi yelp clf; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_emit|k_pass1|k_pass2" -s 9 -c 3 -o $O/full_$c python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_full_$c.log 2>&1; echo ncu-full $c rc=$?
done
timeout 900 python scripts/size_sweep.py yelp taxi > $O/size_sweep.jsonl 2>&1; echo sweep rc=$?
