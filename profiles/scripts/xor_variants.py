"""(Experiment record: variant 9 was a temporary make_variant<32, 8, 13, 1>
instantiation, removed after this measurement.)
Fused XOR checksum of 2^34 words at L=32 (the bench's e2e_xor call) by
kernel variant: 7 = 8-lane groups, two lanes per thread (the default for the
fused mode); 9 = 8-lane groups, one lane per thread (twice the warps);
0 = the store-mode default shape. ms per call (8 calls after 3 warm-up)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2309_16682_b200 as V  # noqa: E402

n = 1 << 34
for variant in (0, 9, 0, 9):
    g = V.VmtGenerator(5489, V.VmtConfig(32))
    g.set_tuning(variant=variant)
    for _ in range(3):
        g.checksum_xor(n)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(8):
        x = g.checksum_xor(n)
    dt = (time.perf_counter() - t0) / 8
    print(json.dumps({"variant": variant, "ms": round(dt * 1e3, 3), "words_s": round(n / dt / 1e12, 3),
                      "checksum": hex(x)}), flush=True)
