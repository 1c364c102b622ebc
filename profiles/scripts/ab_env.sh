#!/bin/bash
# Environment-switch variants of one library in the driver's bench shape,
# interleaved over ROUNDS on one box.
# Usage: ab_env.sh ROUNDS "VAR=1 VAR2=2" "VAR=2" ... [-- bench args]
R=$1; shift; CFGS=(); while [ $# -gt 0 ] && [ "$1" != "--" ]; do CFGS+=("$1"); shift; done; [ "$1" = "--" ] && shift
OUT=${OUT:-gpurun_out}
for i in $(seq 1 $R); do
  k=0
  for C in "${CFGS[@]}"; do
    k=$((k+1))
    env $C python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-extras "$@" > $OUT/abe_${k}_$i.json 2> $OUT/abe_${k}_$i.err
    python3 -c "
import json
d=json.loads(open('$OUT/abe_${k}_$i.json').read().strip().splitlines()[-1])
t=d['timing_breakdown_ms']
print('[$C]', $i, round(d['ms_per_step'],3), 'gen', round(t['gen_kernel'],3), 'pos', round(t['positioning'],3), 'frac', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks'].get('power_w_median'))"
  done
done
