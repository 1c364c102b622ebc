#!/bin/bash
# Power / clock draw of the generation kernel's parts under sustained load
# (run on the B200 box from the repo root after build.sh): each workload runs
# ~4 s while nvidia-smi samples SM clock, power and throttle reasons every
# 100 ms; prints the workload's own JSON line and the sample medians.
B=profiles/scripts/microbench/_bin
OUT=${OUT:-gpurun_out}
sample() { # name cmd...
  local name=$1; shift
  nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader,nounits -lms 100 > $OUT/pw_$name.csv &
  local smi=$!
  sleep 0.5
  local line; line=$("$@"); [ -z "$line" ] && line="{}"
  kill $smi; wait $smi 2>/dev/null
  python3 - "$name" "$line" $OUT/pw_$name.csv <<'PY'
import sys, json, statistics
name, line, f = sys.argv[1], sys.argv[2], sys.argv[3]
rows = []
for l in open(f):
    r = [x.strip() for x in l.split(",")]
    try: rows.append((float(r[0]), float(r[1]), int(r[2], 16)))
    except Exception: pass
load = [r for r in rows if r[1] > 300] or rows
print(json.dumps({"workload": name, "result": json.loads(line.strip().splitlines()[-1].replace("inf", "null").replace("nan", "null")) if line.strip() else None,
                  "samples_under_load": len(load), "sm_mhz_median": statistics.median(r[0] for r in load),
                  "power_w_median": statistics.median(r[1] for r in load), "power_w_max": max(r[1] for r in load),
                  "reasons_hex": sorted({hex(r[2]) for r in load})}))
PY
}
sample idle sleep 3
sample stg64_rand $B/probe_power stg64 1400
sample stg128_rand $B/probe_power stg128 1500
sample tma_bulk_1 $B/probe_power tma 1500 1
sample tma_bulk_2 $B/probe_power tma 1500 2
sample tma_bulk_4 $B/probe_power tma 1500 4
sample gen_store env MB_ONLY=store $B/mb_base 1300
sample gen_compute_only env MB_ONLY=xor $B/mb_base 1600
sample store_probe_v2 $B/probe_st 1400 v2
sample store_probe_v4 $B/probe_st 1400 v4
sample gen_inplace $B/inplace 1300
sample gen_inplace_tma $B/inplace_tma 1300
