"""Short-run kernel shapes for the 8- and 16-lane fills (variants 9-11: runs of
4 or 8 words, one lane per thread -> 416-832 threads per chunk instead of
128): device time per fill (CUDA events, 20 fills after 8 warm-up fills) by
variant and chunk count, config 2 (L=8, 2^28 values) and config 1 (L=16, 2^26
words). Every variant's stream is checked against variant 0's XOR checksum of
the same fill. Run on the B200 box from the repo root.

Variants 9-11 were measured slower (profiles/r02_short_run_sweep.log) and are
not instantiated in the product library; to repeat the run add translation
units with
  L=8 : make_variant<8, 8, 4, 1>(9), make_variant<8, 8, 8, 1>(10)
  L=16: make_variant<16, 16, 8, 1>(9), make_variant<16, 16, 4, 2>(10), make_variant<16, 16, 4, 1>(11)
to csrc/ (like variants_l8.cu), list them in build.py SOURCES and in
pick_variant (vmt_capi.cu)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2309_16682_b200 as V  # noqa: E402


def xor_of(t):
    x = t.view(torch.int32)
    while x.numel() > 1 << 20:
        h = x.numel() // 2
        x = x[:h] ^ x[h:2 * h]
    r = 0
    for v in x.cpu().numpy().view("uint32"):
        r ^= int(v)
    return r


def sweep(L, seed, n, kinds, variants, chunk_list):
    ref = {}
    for kind in kinds:
        dt = {"f32": torch.float32, "f64": torch.float64, "u32": torch.uint32}[kind]
        buf = torch.empty(n, dtype=dt, device="cuda")
        for variant in variants:
            for chunks in chunk_list:
                g = V.VmtGenerator(seed, V.VmtConfig(L))
                g.set_tuning(max_chunks=chunks, variant=variant)
                fill = {"f32": g.fill_f32, "f64": g.fill_f64, "u32": g.fill_u32}[kind]
                for _ in range(8):
                    fill(buf)
                torch.cuda.synchronize()
                g.set_profiling(True)
                g.profile_totals()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(20):
                    fill(buf)
                e1.record()
                e1.synchronize()
                fills, jump, gen = g.profile_totals()
                g.set_profiling(False)
                # the 28th fill's content, identical for every shape
                x = xor_of(buf if kind != "f64" else buf.view(torch.int64).to(torch.int32))
                ref.setdefault(kind, x)
                print(json.dumps({"L": L, "kind": kind, "variant": variant, "chunks": chunks,
                                  "ms": round(e0.elapsed_time(e1) / 20, 4), "gen_ms": round(gen / max(fills, 1), 4),
                                  "pos_wait_ms": round(jump / max(fills, 1), 4), "same": x == ref[kind]}), flush=True)
                del g
        del buf


which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "c2"):
    sweep(8, 42, 1 << 28, ("f32", "f64", "u32"), (0, 9, 10), (0, 74, 100, 148, 296))
if which in ("all", "c1"):
    sweep(16, 5489, 1 << 26, ("u32",), (0, 9, 10, 11), (0, 37, 50, 64, 75, 100, 148))
