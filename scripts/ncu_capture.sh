# One ncu --set full capture of the bench's exact launch (the full qwen7b batch) for the roofline traffic,
# plus the launch list of the bench command. Run on the GPU box: gpurun -- bash scripts/ncu_capture.sh
O=gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_score|k_compact|k_select" -c 3 \
  -o $O/prof_full -f python scripts/profile_step.py --requests 64 > $O/prof_full.log 2>&1
ncu -i $O/prof_full.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active > $O/prof_full_raw.csv 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/launches_bench.log 2>&1
