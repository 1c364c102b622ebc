"""Config 1 (L=16, 2^26 words per fill, consecutive fills) by kernel variant
and chunk count: device time per fill (CUDA events, 20 fills after 8 warm-up
fills), to find what bounds it. Run on the B200 box from the repo root."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2309_16682_b200 as V  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 16
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 26
buf = torch.empty(n, dtype=torch.uint32, device="cuda")
for variant in (0, 4):
    for chunks in (0, 24, 37, 50, 64, 75, 100, 148, 296):
        g = V.VmtGenerator(5489, V.VmtConfig(L))
        g.set_tuning(max_chunks=chunks, variant=variant)
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
        print(json.dumps({"L": L, "n": n, "variant": variant, "max_chunks": chunks, "ms": round(ms, 4),
                          "gen_ms": round(gen / max(fills, 1), 4), "pos_wait_ms": round(jump / max(fills, 1), 4),
                          "tbs": round(n * 4 / ms / 1e9, 3), "prefetch": g.prefetch_stats()}), flush=True)
        del g
