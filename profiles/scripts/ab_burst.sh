#!/bin/bash
# Burst shape (the bench default: 3 warm-up + 5 steps, with the other configs)
# for several library builds, interleaved. Usage: ab_burst.sh ROUNDS LIB...
R=$1; shift; OUT=${OUT:-gpurun_out}
for i in $(seq 1 $R); do
  for L in "$@"; do
    tag=$(basename $L .so)
    VMT_LIB=$L python bench.py --no-e2e --no-cpu-baseline > $OUT/abb_${tag}_$i.json 2> $OUT/abb_${tag}_$i.err
    python3 -c "
import json
d=json.loads(open('$OUT/abb_${tag}_$i.json').read().strip().splitlines()[-1])
oc={k:round(v.get('ms',0),3) for k,v in d.get('other_configs',{}).items() if isinstance(v,dict)}
print('$tag', $i, round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], oc, d['roofline']['store_probe'])"
  done
done
