cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_emit -s 3 -c 1 -o gpurun_out/prof_emit_ts python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --timestamps --records 5000000 > gpurun_out/ncu_ts.log 2>&1; echo ncu rc=$?
