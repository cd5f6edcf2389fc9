# usage (GPU box): bash scripts/gpu_prof_r2.sh <tag> [configs...] -> gpurun_out/<tag>/: ncu --set full of
# k_pass1 / k_pass2 / k_emit per config (reduced records), SASS-level source pages, summaries.
cd $GRAFT_REPO_ROOT
tag=$1; shift
O=gpurun_out/$tag; mkdir -p $O
for c in "$@"; do
  recs=${RECS:-1000000}; [ "$c" = taxi ] && recs=${RECS_TAXI:-8000000}; [ "$c" = clf ] && recs=${RECS_CLF:-8000000}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KRE:-k_emit|k_pass1|k_pass2}" -s ${SKIP:-9} -c ${CNT:-3} \
    -o $O/full_$c python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu --records $recs > $O/ncu_$c.log 2>&1
  echo "ncu $c rc=$?"
  ncu -i $O/full_$c.ncu-rep --page source --csv --print-source sass > $O/sass_$c.csv 2>/dev/null
  ncu -i $O/full_$c.ncu-rep --page raw --csv > $O/raw_$c.csv 2>/dev/null
done
ls -la $O
