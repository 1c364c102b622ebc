#!/bin/bash
# A/B of two builds of the library on ONE box (boxes differ by several % in
# sustained power-capped rate): driver-shaped benches (20 steps, 5 warm-up)
# interleaved. Usage: ab_bench.sh LIB_A LIB_B [rounds] [extra bench args]
A=$1; B=$2; N=${3:-2}; shift 3; OUT=${OUT:-gpurun_out}
for i in $(seq 1 $N); do
  for L in $A $B; do
    tag=$(basename $L .so)
    VMT_LIB=$L python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline "$@" > $OUT/ab_${tag}_$i.json 2> $OUT/ab_${tag}_$i.err
    python3 -c "
import json,sys
d=json.loads(open('$OUT/ab_${tag}_$i.json').read().strip().splitlines()[-1])
oc={k:round(v.get('ms',0),3) for k,v in d.get('other_configs',{}).items() if isinstance(v,dict)}
print('$tag', $i, round(d['ms_per_step'],3), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['samples'], d['clocks'].get('power_w_median'), d['checksum_xor']==d['checksum_oracle'], oc)"
  done
done
