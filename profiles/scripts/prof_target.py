"""Single-launch targets for `ncu --set full` (one kernel of interest per run).

  gen   : vmt_gen_kernel, store mode, L=32 full period, 2^32 words, 148 chunks
          (one chunk per SM, the bench's shape; 2^32 instead of 2^34 so ncu's
          save/restore of the written buffer stays at 16 GiB)
  jump  : vmt_jump_kernel, the bench's positioning launch (147 x 32 = 4704 jobs)
  stats : vmt_gen_kernel MODE_STATS (fused monobit + byte histogram), 2^32 words
  xor   : vmt_gen_kernel MODE_XOR (fused checksum), 2^32 words
  posmma: vmt_posmma2_kernel, the co-resident tcgen05 FP4 positioning GEMM (CTA pairs)
          (4736 lane states x F^(624 D)); under ncu it runs serialised, i.e.
          alone on the GPU (6 fills of 2^32 words; it launches from fill 3 on)
  steady: the bench's steady state -- 2^34-word fills at L=32 with the
          co-resident positioning prefetch; the 9th fill is bracketed by
          cudaProfilerStart/Stop so `ncu --replay-mode app-range
          --profile-from-start off` measures ONE whole step (generation kernel
          + the next step's tcgen05 positioning GEMM running beside it)
          with the kernels concurrent, as in the bench
  c5    : config 5 as bench.py runs it (4096 seeded states, 64-bit jumps), 3 calls
  c1/c2/c3: the other BASELINE configs as bench.py's extras run them (8
          repeats of each call, past the one-time matrix builds) -- for the
          launch lists showing every kernel is ours
Each target runs its call three times; profile with --launch-skip/-c on the
kernel name (see profiles/scripts/profile.sh).
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2309_16682_b200 as V  # noqa: E402

what = sys.argv[1]
n = 1 << 32
if what == "c5":
    import numpy as np
    seeds = np.arange(1, 4097, dtype=np.uint32)
    states = torch.from_numpy(V.seed_states(seeds).view(np.int32)).cuda().view(torch.uint32)
    dists = np.random.default_rng(7).integers(0, 2**63, 4096, dtype=np.int64).view(np.uint64)
    jumped = torch.empty_like(states)
    for _ in range(3):
        V.jump_states(states, dists, out=jumped)
    torch.cuda.synchronize()
    print("done", what)
    sys.exit(0)
if what == "steady":
    g = V.VmtGenerator(5489, V.VmtConfig(32))
    buf = torch.empty(1 << 34, dtype=torch.uint32, device="cuda")
    for _ in range(8):
        g.fill_u32(buf)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    g.fill_u32(buf)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    st = g.prefetch_stats()
    assert st["tensor_prefetches"] >= 6, st
    print("done", what, st)
    sys.exit(0)
if what in ("c1", "c2", "c3"):
    if what == "c1":
        g = V.VmtGenerator(5489, V.VmtConfig(16))
        b = torch.empty(1 << 26, dtype=torch.uint32, device="cuda")
        for _ in range(8):
            g.fill_u32(b)
    elif what == "c2":
        g = V.VmtGenerator(42, V.VmtConfig(8))
        f = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
        d = torch.empty(1 << 28, dtype=torch.float64, device="cuda")
        for _ in range(8):
            g.fill_f32(f)
        for _ in range(8):
            g.fill_f64(d)
    else:
        b = torch.empty(1024 << 20, dtype=torch.uint32, device="cuda")
        for _ in range(4):
            V.batch_fill_u32(b, 1, 1024, 16, 1 << 20)
    torch.cuda.synchronize()
    print("done", what)
    sys.exit(0)
g = V.VmtGenerator(5489, V.VmtConfig(32))
g.set_tuning(max_chunks=148)
if what in ("gen", "jump"):
    buf = torch.empty(n, dtype=torch.uint32, device="cuda")
    for _ in range(3):
        g.fill_u32(buf)
elif what == "stats":
    for _ in range(3):
        g.stat_counts(n)
elif what == "posmma":
    g.set_prefetch(2)
    buf = torch.empty(n, dtype=torch.uint32, device="cuda")
    for _ in range(6):
        g.fill_u32(buf)
    assert g.prefetch_stats()["tensor_prefetches"] >= 2, g.prefetch_stats()
elif what == "xor":
    for _ in range(3):
        g.checksum_xor(n)
torch.cuda.synchronize()
print("done", what)
