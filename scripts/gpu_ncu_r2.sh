# Round-2 evidence part B: one ncu --set full capture of k_pass1 / k_pass2 / k_emit per workload (reduced
# record counts so the reports stay small), k_small on cfg1; text summaries written on the box (the
# reports themselves are deleted unless KEEP=1).
cd $GRAFT_REPO_ROOT
O=gpurun_out/ncu2; mkdir -p $O
for c in yelp taxi clf; do
  recs=1000000; [ $c = taxi ] && recs=8000000; [ $c = clf ] && recs=8000000
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_emit|k_pass1|k_pass2" -s 9 -c 3 \
    -o $O/full_$c python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu --parity none --records $recs > $O/ncu_full_$c.log 2>&1; echo ncu-full $c rc=$?
  for k in k_pass1 k_pass2 k_emit; do
    ncu -i $O/full_$c.ncu-rep -k regex:$k --page raw --csv > $O/raw_${c}_$k.csv 2>/dev/null
    python scripts/stall_lines.py $O/full_$c.ncu-rep $k 20 > $O/stall_${c}_$k.txt 2>&1
    python scripts/src_hot.py $O/full_$c.ncu-rep $k 25 > $O/hot_${c}_$k.txt 2>&1
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_small" -s 5 -c 1 \
  -o $O/full_cfg1 python bench.py --config cfg1 --steps 1 --warmup 3 --no-e2e --no-cpu --no-graph --parity none > $O/ncu_full_cfg1.log 2>&1; echo ncu-full cfg1 rc=$?
ncu -i $O/full_cfg1.ncu-rep --page raw --csv > $O/raw_cfg1_k_small.csv 2>/dev/null
python scripts/stall_lines.py $O/full_cfg1.ncu-rep k_small 20 > $O/stall_cfg1_k_small.txt 2>&1
[ -z "$KEEP" ] && rm -f $O/*.ncu-rep
du -sh $O; ls $O | head -50
