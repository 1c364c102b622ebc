"""Randomised stress of the steady-state positioning (GEMM prefetch with the
dynamic tile scheduler, operand ahead / side stream, block advance, shape
changes, skips, several generators interleaved): every fill word-identical to
a generator positioned by polynomial jumps only. usage: stress_positioning.py [fills] [seed]"""
import random
import sys

import torch

sys.path.insert(0, ".")
import paper_2309_16682_b200 as V  # noqa: E402

fills = int(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
gens = []
for L, seed in ((32, 5), (16, 6), (8, 7), (16, 8)):
    ref = V.VmtGenerator(seed, V.VmtConfig(L))
    ref.set_positioning(1)
    ref.set_prefetch(0)
    tst = V.VmtGenerator(seed, V.VmtConfig(L))
    gens.append((L, ref, tst))
sizes = [(1 << 24) + 17, 1 << 25, (1 << 26) + 4096, 3 << 24, 1 << 27]
bufa = torch.empty(max(sizes), dtype=torch.uint32, device="cuda")
bufb = torch.empty(max(sizes), dtype=torch.uint32, device="cuda")
cur = [rng.choice(sizes) for _ in gens]
for i in range(fills):
    k = rng.randrange(len(gens))
    L, ref, tst = gens[k]
    r = rng.random()
    if r < 0.08:
        cur[k] = rng.choice(sizes)  # shape change: the prefetched states are discarded
    elif r < 0.12:
        d = rng.randrange(1, 1 << 22)
        ref.skip(d)
        tst.skip(d)
    elif r < 0.16:
        tst.set_tuning(max_chunks=rng.choice([0, 37, 60, 75, 148]))
        ref.set_tuning(max_chunks=rng.choice([0, 37, 148]))
    n = cur[k]
    ref.fill_u32(bufa[:n])
    tst.fill_u32(bufb[:n])
    if rng.random() < 0.5:
        torch.cuda.synchronize()
    assert torch.equal(bufa[:n].view(torch.int32), bufb[:n].view(torch.int32)), (i, k, L, n)
torch.cuda.synchronize()
print("ok", fills, [(L, t.prefetch_stats(), t.positioning_stats()) for L, _, t in gens])
