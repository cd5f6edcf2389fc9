cd $GRAFT_REPO_ROOT
for w in yelp taxi clf; do timeout 120 python scripts/probe2.py $w 2e9 2>&1 | grep -E "GB|Error" | tail -3; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_scan -s 2 -c 1 -o gpurun_out/prof_yelp_v5 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config yelp --records 1400000 > gpurun_out/ncu_yelp_v5.log 2>&1; echo ncu rc=$?
