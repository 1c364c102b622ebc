"""L=16 fills (config 1's 2^26 words and 2^28) by kernel variant (0 = R13 VW2
default, 4 = R13 VW1: twice the threads per chunk) and chunk count: device
ms per fill (20 fills after 8 warm-up fills)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2309_16682_b200 as V  # noqa: E402

for n in (1 << 26, 1 << 28):
    buf = torch.empty(n, dtype=torch.uint32, device="cuda")
    for variant in (0, 4):
        for chunks in (0, 64, 75, 100, 148, 296):
            g = V.VmtGenerator(5489, V.VmtConfig(16))
            g.set_tuning(max_chunks=chunks, variant=variant)
            for _ in range(8):
                g.fill_u32(buf)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                g.fill_u32(buf)
            e1.record()
            e1.synchronize()
            print(json.dumps({"n": n, "variant": variant, "chunks": chunks,
                              "ms": round(e0.elapsed_time(e1) / 20, 4)}), flush=True)
            del g
    del buf
