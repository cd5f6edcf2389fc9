# Round-2 final evidence on one B200 (gpurun): smoke, GPU tests, the default bench line (yelp + taxi / clf /
# cfg1 sub-records with full parity), the reference arm, ncu launch lists of the yelp and taxi bench commands,
# taxi64, one ncu --set full capture of k_pass1 / k_pass2 / k_emit per workload (+ k_small on cfg1) with
# per-line summaries, and the rate-vs-size sweep.
cd $GRAFT_REPO_ROOT
O=gpurun_out/final; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -1 $O/smoke.log
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > $O/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 $O/pytest_gpu.log
timeout 1500 python bench.py > $O/bench_default.log 2> $O/bench_default.err; echo bench rc=$?
timeout 900 python bench.py --impl reference > $O/bench_reference.log 2>&1; echo ref rc=$?
for c in yelp taxi; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu --parity none > $O/ncu_launch_$c.log 2>&1; echo ncu-launch $c rc=$?
done
timeout 1200 python bench.py --config taxi64 --steps 3 --warmup 1 > $O/bench_taxi64.log 2> $O/bench_taxi64.err; echo taxi64 rc=$?
for c in yelp taxi clf; do
  recs=1000000; [ $c = taxi ] && recs=8000000; [ $c = clf ] && recs=8000000
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_emit|k_pass1|k_pass2" -s 9 -c 3 \
    -o $O/full_$c python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu --parity none --records $recs > $O/ncu_full_$c.log 2>&1; echo ncu-full $c rc=$?
  for k in k_pass1 k_pass2 k_emit; do
    ncu -i $O/full_$c.ncu-rep -k regex:$k --page raw --csv > $O/raw_${c}_$k.csv 2>/dev/null
    python scripts/src_hot.py $O/full_$c.ncu-rep $k 40 > $O/hot_${c}_$k.txt 2>&1
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_small" -s 5 -c 1 \
  -o $O/full_cfg1 python bench.py --config cfg1 --steps 1 --warmup 3 --no-e2e --no-cpu --no-graph --parity none > $O/ncu_full_cfg1.log 2>&1; echo ncu-full cfg1 rc=$?
ncu -i $O/full_cfg1.ncu-rep --page raw --csv > $O/raw_cfg1_k_small.csv 2>/dev/null
rm -f $O/*.ncu-rep
timeout 900 python scripts/size_sweep.py yelp taxi > $O/size_sweep.jsonl 2> $O/size_sweep.err; echo sweep rc=$?
du -sh $O
