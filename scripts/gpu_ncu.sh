cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_scan -s 2 -c 1 -o gpurun_out/prof_yelp_v4 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config yelp --records 1400000 > gpurun_out/ncu_yelp_v4.log 2>&1; echo ncu rc=$?
