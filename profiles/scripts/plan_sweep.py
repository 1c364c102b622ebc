"""Repeated same-size fills at L = 16 / 32 for several sizes: the planner's
chunk count (max_chunks=0) against fixed ones; device ms per fill (10 fills
after 6 warm-up fills). Finds fill shapes the planner gets wrong."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2309_16682_b200 as V  # noqa: E402

for L in (16, 32):
    for lg in (24, 26, 28, 30, 32):
        n = 1 << lg
        buf = torch.empty(n, dtype=torch.uint32, device="cuda")
        row = {"L": L, "log2n": lg}
        for chunks in (0, 37, 75, 148, 296):
            g = V.VmtGenerator(5489, V.VmtConfig(L))
            g.set_tuning(max_chunks=chunks)
            for _ in range(6):
                g.fill_u32(buf)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                g.fill_u32(buf)
            e1.record()
            e1.synchronize()
            row[str(chunks)] = round(e0.elapsed_time(e1) / 10, 4)
            del g
        print(json.dumps(row), flush=True)
        del buf
