import sys, time, torch
sys.path.insert(0, ".")
import paper_2309_16682_b200 as V
buf = torch.empty(1 << 20, dtype=torch.uint32, device="cuda")
for L in (32, 16, 8, 1):
    for rep in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        g = V.VmtGenerator(1000 + rep, V.VmtConfig(L))
        torch.cuda.synchronize(); t1 = time.perf_counter()
        g.fill_u32(buf)
        torch.cuda.synchronize(); t2 = time.perf_counter()
        x = g.next_u32() if hasattr(g, "next_u32") else None
        t3 = time.perf_counter()
        print(L, rep, "create ms", round((t1 - t0) * 1e3, 3), "first fill 2^20 ms", round((t2 - t1) * 1e3, 3), "next_u32 ms", round((t3 - t2) * 1e3, 3), flush=True)
        del g
