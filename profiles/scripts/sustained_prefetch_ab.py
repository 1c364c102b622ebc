"""Co-resident (prefetch 2) vs serial (prefetch 0) positioning under sustained
load: 2^34-word fills at L=32 in one process, the mode alternating every 20
fills for several rounds (no idle gaps: the board stays at its power cap), device
ms per fill per block of 20. usage: sustained_prefetch_ab.py [rounds]"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2309_16682_b200 as V  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 4
g = V.VmtGenerator(5489, V.VmtConfig(32))
buf = torch.empty(1 << 34, dtype=torch.uint32, device="cuda")
for _ in range(6):
    g.fill_u32(buf)
res = {0: [], 2: []}
for r in range(rounds):
    for pf in (2, 0):
        g.set_prefetch(pf)
        for _ in range(3):
            g.fill_u32(buf)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            g.fill_u32(buf)
        e1.record()
        e1.synchronize()
        res[pf].append(round(e0.elapsed_time(e1) / 20, 3))
print(json.dumps({"ms_per_fill_prefetch2": res[2], "ms_per_fill_prefetch0": res[0]}))
