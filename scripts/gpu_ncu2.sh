cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python -m pytest tests/test_gpu_parity.py -q -x --timeout 60 2>&1 | tail -2
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_scan -s 2 -c 1 -o gpurun_out/prof_taxi_v6 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config taxi --records 10000000 > gpurun_out/ncu_taxi_v6.log 2>&1; echo ncu rc=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_scan -s 2 -c 1 -o gpurun_out/prof_yelp_v6 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config yelp --records 1400000 > gpurun_out/ncu_yelp_v6.log 2>&1; echo ncu rc=$?
for w in yelp taxi clf; do timeout 120 python scripts/probe2.py $w 2e9 2>&1 | grep -E "fused|Error" | tail -1; done
