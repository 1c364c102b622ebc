OUT=gpurun_out
set -x
for c in c1 c2 c3; do
  python profiles/scripts/prof_target.py $c || exit 1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/s5_launches_$c.csv python profiles/scripts/prof_target.py $c > $OUT/s5_ncu_$c.log 2>&1
done
python profiles/scripts/prof_target.py posmma || exit 1
ncu --set full --clock-control none --import-source on -k regex:vmt_posmma2_kernel --launch-skip 1 -c 1 -o $OUT/s5_prof_posmma -f python profiles/scripts/prof_target.py posmma > $OUT/s5_ncu_posmma.log 2>&1
ncu -i $OUT/s5_prof_posmma.ncu-rep --page details --csv > $OUT/s5_ncu_posmma_details.csv 2>/dev/null
ncu -i $OUT/s5_prof_posmma.ncu-rep --page raw --csv > $OUT/s5_ncu_posmma_raw.csv 2>/dev/null
ls -la $OUT | tail -12
