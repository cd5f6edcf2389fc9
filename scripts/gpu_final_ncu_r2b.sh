cd $GRAFT_REPO_ROOT
O=gpurun_out/final; mkdir -p $O
for c in taxi clf; do
  recs=8000000
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^k_emit$|k_pass1|k_pass2" -s 9 -c 3 \
    -o $O/full_$c python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu --parity none --records $recs > $O/ncu_full_$c.log 2>&1; echo ncu-full $c rc=$?
  for k in k_pass1 k_pass2 "^k_emit$"; do
    kn=$(echo $k | tr -d '^$')
    ncu -i $O/full_$c.ncu-rep -k regex:"$k" --page raw --csv > $O/raw_${c}_$kn.csv 2>/dev/null
    python scripts/src_hot.py $O/full_$c.ncu-rep "$k" 40 > $O/hot_${c}_$kn.txt 2>&1
  done
done
rm -f $O/*.ncu-rep
