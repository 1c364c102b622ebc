"""Per-fill device time, prefetch and matrix-cache counters of repeated
same-size fills (VMT_DEBUG=1 also prints the planner's choice).
Usage: plan_debug.py L log2n [fills]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2309_16682_b200 as V  # noqa: E402

L, lg = int(sys.argv[1]), int(sys.argv[2])
fills = int(sys.argv[3]) if len(sys.argv) > 3 else 20
n = 1 << lg
buf = torch.empty(n, dtype=torch.uint32, device="cuda")
g = V.VmtGenerator(5489, V.VmtConfig(L))
for i in range(fills):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.fill_u32(buf)
    e1.record()
    e1.synchronize()
    print("fill", i, round(e0.elapsed_time(e1), 3), g.prefetch_stats(), g.positioning_stats(), flush=True)
