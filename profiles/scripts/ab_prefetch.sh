#!/bin/bash
# Co-resident tcgen05 positioning (prefetch 2) vs serial positioning
# (prefetch 0) in the driver's bench shape, interleaved on one box.
OUT=${OUT:-gpurun_out}
for i in 1 2 3; do
  for pf in 2 0; do
    python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-extras --prefetch $pf > $OUT/abpf_${pf}_$i.json 2> $OUT/abpf_${pf}_$i.err
    python3 -c "
import json
d=json.loads(open('$OUT/abpf_${pf}_$i.json').read().strip().splitlines()[-1])
t=d['timing_breakdown_ms']
print('prefetch=$pf', $i, round(d['ms_per_step'],3), 'gen', round(t['gen_kernel'],3), 'pos', round(t['positioning'],3), 'frac', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['samples'], d['clocks'].get('reasons'))"
  done
done
