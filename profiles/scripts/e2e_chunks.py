"""End-to-end fill into pinned host memory (16 GiB per call) by the chunk
count of the generation launches: does the generation kernel's HBM traffic
slow the concurrent D2H copies? Plain pinned memcpy of the same size beside it."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2309_16682_b200 as V  # noqa: E402

n = 1 << 32
host = torch.empty(n, dtype=torch.uint32, pin_memory=True)
src = torch.empty(1 << 28, dtype=torch.uint32, device="cuda")
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(16):
        host[k << 28:(k + 1) << 28].copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    print(json.dumps({"memcpy_gbs": round(n * 4 / (time.perf_counter() - t0) / 1e9, 2)}), flush=True)
for chunks in [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "0,74,37,18,9,0").split(",")]:
    g = V.VmtGenerator(5489, V.VmtConfig(32))
    g.set_tuning(max_chunks=chunks)
    g.fill_u32(host)
    t0 = time.perf_counter()
    for _ in range(2):
        g.fill_u32(host)
    dt = (time.perf_counter() - t0) / 2
    print(json.dumps({"max_chunks": chunks, "gbs": round(n * 4 / dt / 1e9, 2)}), flush=True)
    del g
