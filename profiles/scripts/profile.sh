#!/bin/bash
# Captures the committed profiles (run on the B200 box from the repo root):
#   launch list of the bench command (cold, serialised; shares only)
#   ncu --set full of the top kernels, one launch each
set -x
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-extras > $OUT/bench_plain.json || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-extras > $OUT/ncu_launches.log 2>&1
for t in gen stats xor; do
  python profiles/scripts/prof_target.py $t || exit 1
  ncu --set full --clock-control none --import-source on -k regex:vmt_gen_kernel --launch-skip 2 -c 1 \
      -o $OUT/prof_$t -f python profiles/scripts/prof_target.py $t > $OUT/ncu_$t.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:vmt_jump_kernel --launch-skip 2 -c 1 \
    -o $OUT/prof_jump -f python profiles/scripts/prof_target.py jump > $OUT/ncu_jump.log 2>&1
python profiles/scripts/prof_target.py posmma || exit 1
ncu --set full --clock-control none --import-source on -k regex:vmt_posmma --launch-skip 1 -c 1 \
    -o $OUT/prof_posmma -f python profiles/scripts/prof_target.py posmma > $OUT/ncu_posmma.log 2>&1
ls -la $OUT
