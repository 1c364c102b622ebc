"""Config 2 (L=8, seed 42, 2^28 float32 / float64 per fill, consecutive fills):
device time per fill by chunk count, 3 repetitions each (20 fills after 8
warm-up fills), to see what bounds it and how much it varies."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2309_16682_b200 as V  # noqa: E402

n = 1 << 28
for kind in ("f32", "f64"):
    buf = torch.empty(n, dtype=torch.float32 if kind == "f32" else torch.float64, device="cuda")
    for chunks in (0, 148, 222, 296, 444):
        for rep in range(3):
            g = V.VmtGenerator(42, V.VmtConfig(8))
            g.set_tuning(max_chunks=chunks)
            fill = g.fill_f32 if kind == "f32" else g.fill_f64
            for _ in range(8):
                fill(buf)
            torch.cuda.synchronize()
            g.set_profiling(True)
            g.profile_totals()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                fill(buf)
            e1.record()
            e1.synchronize()
            fills, jump, gen = g.profile_totals()
            g.set_profiling(False)
            ms = e0.elapsed_time(e1) / 20
            print(json.dumps({"kind": kind, "max_chunks": chunks, "rep": rep, "ms": round(ms, 4),
                              "gen_ms": round(gen / max(fills, 1), 4), "pos_wait_ms": round(jump / max(fills, 1), 4),
                              "gbs": round(n * buf.element_size() / ms / 1e6, 1), "prefetch": g.prefetch_stats()}),
                  flush=True)
            del g
    del buf
