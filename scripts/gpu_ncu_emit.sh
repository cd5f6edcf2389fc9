# usage (GPU box): bash scripts/gpu_ncu_emit.sh [config] [tag]  -> gpurun_out/prof_emit_<tag>.ncu-rep + SASS csv
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cfg=${1:-taxi}; tag=${2:-$cfg}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_emit -s 3 -c 1 -o gpurun_out/prof_emit_$tag python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e --no-cpu --records ${RECS:-5000000} > gpurun_out/ncu_emit_$tag.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/prof_emit_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_emit_$tag.csv 2>/dev/null; echo sass rc=$?
