# Round-2 evidence on one B200 (run under gpurun), part A: smoke, GPU tests, the default bench line
# (yelp + taxi / clf / cfg1 sub-records, full parity), the reference arm, the ncu launch lists of the
# yelp and taxi bench commands, and the 64 GB taxi64 run.
cd $GRAFT_REPO_ROOT
O=gpurun_out/ev2; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -1 $O/smoke.log
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > $O/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 $O/pytest_gpu.log
timeout 1500 python bench.py > $O/bench_default.log 2> $O/bench_default.err; echo bench rc=$?
timeout 900 python bench.py --impl reference > $O/bench_reference.log 2>&1; echo ref rc=$?
for c in yelp taxi; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu --parity none > $O/ncu_launch_$c.log 2>&1; echo ncu-launch $c rc=$?
done
timeout 1200 python bench.py --config taxi64 --steps 3 --warmup 1 > $O/bench_taxi64.log 2> $O/bench_taxi64.err; echo taxi64 rc=$?
du -sh $O; ls -la $O
