cd $GRAFT_REPO_ROOT
O=gpurun_out/ps; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_emit_sparse" -s 3 -c 1 \
  -o $O/full_yelp python bench.py --config yelp --steps 1 --warmup 3 --no-e2e --no-cpu --parity none --records 1000000 > $O/ncu.log 2>&1; echo ncu rc=$?
python scripts/src_hot.py $O/full_yelp.ncu-rep k_emit_sparse 60 > $O/hot.txt 2>&1
python scripts/stall_lines.py $O/full_yelp.ncu-rep k_emit_sparse 25 > $O/stall.txt 2>&1
ncu -i $O/full_yelp.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
rm -f $O/*.ncu-rep
