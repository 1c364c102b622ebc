#!/bin/bash
# Several library builds in the driver's bench shape (20 steps / 5 warm-up),
# interleaved over ROUNDS on one box. Usage: ab_libs.sh ROUNDS LIB... [-- bench args]
R=$1; shift; LIBS=(); while [ $# -gt 0 ] && [ "$1" != "--" ]; do LIBS+=("$1"); shift; done; [ "$1" = "--" ] && shift
OUT=${OUT:-gpurun_out}
for i in $(seq 1 $R); do
  for L in "${LIBS[@]}"; do
    tag=$(basename $L .so)
    VMT_LIB=$L python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-extras "$@" > $OUT/abl_${tag}_$i.json 2> $OUT/abl_${tag}_$i.err
    python3 -c "
import json
d=json.loads(open('$OUT/abl_${tag}_$i.json').read().strip().splitlines()[-1])
t=d['timing_breakdown_ms']
print('$tag', $i, round(d['ms_per_step'],3), 'gen', round(t['gen_kernel'],3), 'pos', round(t['positioning'],3), 'frac', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['samples'], d['clocks'].get('power_w_median'))"
  done
done
