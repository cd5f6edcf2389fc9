# per-source-line instruction accounting (all lines) of k_emit / k_pass2 on yelp and taxi (reduced sizes)
cd $GRAFT_REPO_ROOT
O=gpurun_out/lines; mkdir -p $O
for c in yelp taxi; do
  recs=1000000; [ $c = taxi ] && recs=8000000
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_emit|k_pass2" -s 6 -c 2 \
    -o $O/full_$c python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu --parity none --records $recs > $O/ncu_$c.log 2>&1; echo ncu $c rc=$?
  for k in k_pass2 k_emit; do python scripts/src_hot.py $O/full_$c.ncu-rep $k 400 > $O/lines_${c}_$k.txt 2>&1; done
done
rm -f $O/*.ncu-rep
