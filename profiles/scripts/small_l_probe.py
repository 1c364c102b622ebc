"""What bounds the 8/16-lane store fills: the same fill in store mode and as a
fused XOR (no stores), by kernel variant, at a fixed chunk count. Device time
per fill (CUDA events, 20 fills after 8 warm-up fills)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2309_16682_b200 as V  # noqa: E402

for L, seed, n, variants, chunk_list in ((8, 42, 1 << 28, (3, 4, 5, 1), (148,)), (16, 5489, 1 << 26, (3, 4, 5, 1), (75,)),
                                         (32, 5489, 1 << 28, (3, 4), (148,))):
    buf = torch.empty(n, dtype=torch.uint32, device="cuda")
    for variant in variants:
        for chunks in chunk_list:
            for mode in ("u32", "xor"):
                g = V.VmtGenerator(seed, V.VmtConfig(L))
                g.set_tuning(max_chunks=chunks, variant=variant)
                fn = (lambda: g.fill_u32(buf)) if mode == "u32" else (lambda: g.checksum_xor(n))
                for _ in range(8):
                    fn()
                torch.cuda.synchronize()
                g.set_profiling(True)
                g.profile_totals()
                for _ in range(20):
                    fn()
                torch.cuda.synchronize()
                fills, jump, gen = g.profile_totals()
                print(json.dumps({"L": L, "variant": variant, "chunks": chunks, "mode": mode,
                                  "gen_ms": round(gen / max(fills, 1), 4), "pos_ms": round(jump / max(fills, 1), 4)}),
                      flush=True)
                del g
