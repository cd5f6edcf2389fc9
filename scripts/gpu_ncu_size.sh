# k_emit memory counters at two input sizes (taxi; 10 M and 48.9 M records), one ncu pass set each
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_op_write_hit_rate.pct,lts__t_sector_op_read_hit_rate.pct,smsp__inst_executed.sum
for R in 10000000 48900000; do
timeout 1200 ncu --metrics $M --clock-control none -k regex:k_emit -s 3 -c 1 --csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --records $R > gpurun_out/emit_mem_$R.csv 2>&1; echo rc=$?
done
