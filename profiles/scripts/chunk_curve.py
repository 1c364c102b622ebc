"""Repeated same-size u32 fills by chunk count and prefetch mode: device ms per
fill with the generation-kernel / positioning-wait split (vmt_profile_totals),
20 fills after 8 warm-up fills. Finer than c1_sweep.py / plan_sweep.py: the
curve the planner's cost model has to follow.
usage: chunk_curve.py L log2n chunks,chunks,... [prefetch modes, default 2,0]"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2309_16682_b200 as V  # noqa: E402

L = int(sys.argv[1])
lg = int(sys.argv[2])
chunk_list = [int(c) for c in sys.argv[3].split(",")]
modes = [int(m) for m in sys.argv[4].split(",")] if len(sys.argv) > 4 else [2, 0]
n = 1 << lg
buf = torch.empty(n, dtype=torch.uint32, device="cuda")
for pf in modes:
    for chunks in chunk_list:
        g = V.VmtGenerator(5489, V.VmtConfig(L))
        g.set_tuning(max_chunks=chunks)
        g.set_prefetch(pf)
        for _ in range(8):
            g.fill_u32(buf)
        torch.cuda.synchronize()
        g.set_profiling(True)
        g.profile_totals()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            g.fill_u32(buf)
        e1.record()
        e1.synchronize()
        fills, jump, gen = g.profile_totals()
        g.set_profiling(False)
        ms = e0.elapsed_time(e1) / 20
        print(json.dumps({"L": L, "log2n": lg, "prefetch": pf, "max_chunks": chunks, "ms": round(ms, 4),
                          "gen_ms": round(gen / max(fills, 1), 4), "pos_ms": round(jump / max(fills, 1), 4),
                          "tbs": round(n * 4 / ms / 1e9, 3), "pf": g.prefetch_stats()}), flush=True)
        del g
