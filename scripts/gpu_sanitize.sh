# compute-sanitizer sweep of the GPU tests (run under gpurun): memcheck on every GPU test file, racecheck
# on the parity tests of every workload (shared-memory hazards of the warp-level emission), synccheck.
cd $GRAFT_REPO_ROOT
timeout 1500 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ranges.py tests/test_gpu_scale.py -q -x 2>&1 | tail -3
timeout 900 compute-sanitizer --tool racecheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -q -x -k "smoke or cfg1 or fixtures or yelp or clf or strings or infer" 2>&1 | tail -3
timeout 600 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_parity.py -q -x -k "cfg1" 2>&1 | tail -2
