"""Serial positioning GEMM time by row count: repeated same-size fills with
the prefetch off and GEMM positioning forced, the positioning time per fill
from the profiling events (FP4 operand + GEMM + any block advance).
usage: gemm_rows.py [L chunks]..."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2309_16682_b200 as V  # noqa: E402

shapes = [(16, 16), (16, 32), (16, 64), (16, 75), (16, 80), (32, 74), (32, 148), (16, 512), (16, 1024)]
if len(sys.argv) > 2:
    shapes = [(int(sys.argv[i]), int(sys.argv[i + 1])) for i in range(1, len(sys.argv) - 1, 2)]
for L, chunks in shapes:
    # a whole number of blocks per chunk so no block advance is needed
    n = chunks * 32 * 624 * L
    buf = torch.empty(n, dtype=torch.uint32, device="cuda")
    g = V.VmtGenerator(5489, V.VmtConfig(L))
    g.set_tuning(max_chunks=chunks)
    g.set_prefetch(0)
    g.set_positioning(2)
    for _ in range(8):
        g.fill_u32(buf)
    torch.cuda.synchronize()
    g.set_profiling(True)
    g.profile_totals()
    for _ in range(20):
        g.fill_u32(buf)
    torch.cuda.synchronize()
    fills, jump, gen = g.profile_totals()
    print(json.dumps({"L": L, "chunks": chunks, "rows": L * chunks, "pos_ms": round(jump / fills, 4),
                      "gen_ms": round(gen / fills, 4), "gemms": g.positioning_stats()}), flush=True)
    del g, buf
