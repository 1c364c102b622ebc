#!/bin/bash
# DRAM bytes and duration of one steady-state bench step (app-range replay)
# per library build. Usage: steady_dram.sh LIB...
OUT=${OUT:-gpurun_out}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second
for L in "$@"; do
  tag=$(basename $L .so)
  VMT_LIB=$L ncu --replay-mode app-range --clock-control none --metrics $M --csv --log-file $OUT/sd_$tag.csv \
      python profiles/scripts/prof_target.py steady > $OUT/sd_$tag.log 2>&1
  echo "$tag $(grep -o '"[a-z_.]*","[a-z]*","[0-9.]*"$' $OUT/sd_$tag.csv | tr '\n' ' ')"
done
