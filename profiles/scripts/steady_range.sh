OUT=gpurun_out
M=gpu__time_duration.sum,dram__bytes_write.sum,dram__bytes_read.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second
python profiles/scripts/prof_target.py steady || exit 1
ncu --replay-mode app-range --clock-control none --metrics $M --csv --log-file $OUT/r02_steady_range_ef.csv python profiles/scripts/prof_target.py steady > $OUT/r02_ncu_steady_ef.log 2>&1
grep -o '"[a-z_.]*","[a-z%/]*","[0-9.,]*"$' $OUT/r02_steady_range_ef.csv
