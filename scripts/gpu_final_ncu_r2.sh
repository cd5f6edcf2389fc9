# Round-2 final evidence, part 1 (one B200): ncu launch lists of the yelp and taxi bench commands and one
# ncu --set full capture of k_pass1 / k_pass2 / the emission kernel per workload (+ k_small on cfg1).
cd $GRAFT_REPO_ROOT
O=gpurun_out/final; mkdir -p $O
for c in yelp taxi; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu --parity none > $O/ncu_launch_$c.log 2>&1; echo ncu-launch $c rc=$?
done
for c in yelp taxi clf; do
  recs=1000000; [ $c = taxi ] && recs=8000000; [ $c = clf ] && recs=8000000
  kre="^k_emit$|k_pass1|k_pass2"; [ $c = yelp ] && kre="k_emit_sparse|k_pass1|k_pass2"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$kre" -s 9 -c 3 \
    -o $O/full_$c python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu --parity none --records $recs > $O/ncu_full_$c.log 2>&1; echo ncu-full $c rc=$?
  ke="^k_emit$"; [ $c = yelp ] && ke="k_emit_sparse"
  for k in k_pass1 k_pass2 $ke; do
    kn=$(echo $k | tr -d '^$')
    ncu -i $O/full_$c.ncu-rep -k regex:"$k" --page raw --csv > $O/raw_${c}_$kn.csv 2>/dev/null
    python scripts/src_hot.py $O/full_$c.ncu-rep "$k" 40 > $O/hot_${c}_$kn.txt 2>&1
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_small" -s 5 -c 1 \
  -o $O/full_cfg1 python bench.py --config cfg1 --steps 1 --warmup 3 --no-e2e --no-cpu --no-graph --parity none > $O/ncu_full_cfg1.log 2>&1; echo ncu-full cfg1 rc=$?
ncu -i $O/full_cfg1.ncu-rep --page raw --csv > $O/raw_cfg1_k_small.csv 2>/dev/null
rm -f $O/*.ncu-rep
ls $O
