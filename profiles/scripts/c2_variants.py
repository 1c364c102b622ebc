import json, sys, torch
sys.path.insert(0, ".")
import paper_2309_16682_b200 as V
n = 1 << 28
for kind in ("f32", "f64", "u32"):
    dt = {"f32": torch.float32, "f64": torch.float64, "u32": torch.uint32}[kind]
    buf = torch.empty(n, dtype=dt, device="cuda")
    for variant in (0, 4, 1):
        for chunks in (0, 148, 296, 444):
            g = V.VmtGenerator(42, V.VmtConfig(8))
            g.set_tuning(max_chunks=chunks, variant=variant)
            fill = {"f32": g.fill_f32, "f64": g.fill_f64, "u32": g.fill_u32}[kind]
            for _ in range(8):
                fill(buf)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                fill(buf)
            e1.record(); e1.synchronize()
            print(json.dumps({"kind": kind, "variant": variant, "chunks": chunks, "ms": round(e0.elapsed_time(e1) / 20, 4)}), flush=True)
            del g
    del buf
