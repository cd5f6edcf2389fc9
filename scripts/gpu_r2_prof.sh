# round-2 profiling pass on one B200: GPU tests, then one ncu --set full capture of the pass kernels and k_emit
# on yelp (1 M records) with the SASS source page kept for instruction accounting (scripts/sass_hot.py)
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-p}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > $O/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 $O/pytest_gpu.log
for c in ${CFGS:-yelp}; do
  recs=1000000; [ $c = taxi ] && recs=8000000; [ $c = clf ] && recs=8000000
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KRE:-k_emit|k_pass1|k_pass2}" -s 9 -c 3 \
    -o $O/full_$c python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu --parity none --records $recs > $O/ncu_full_$c.log 2>&1; echo ncu-full $c rc=$?
  for k in k_pass1 k_pass2 k_emit; do
    ncu -i $O/full_$c.ncu-rep -k regex:$k --page raw --csv > $O/raw_${c}_$k.csv 2>/dev/null
    ncu -i $O/full_$c.ncu-rep -k regex:$k --page source --csv --print-source sass > $O/sass_${c}_$k.csv 2>/dev/null
    python scripts/src_hot.py $O/full_$c.ncu-rep $k 25 > $O/hot_${c}_$k.txt 2>&1
  done
done
rm -f $O/*.ncu-rep
