"""Per-CTA timeline of one steady-state fill: the generation kernel and the
co-resident positioning GEMM (start / end in ns on the global timer, SM id),
from a library built with -DVMT_TIMELINE (profiles/scripts/build_ab.sh timeline
"-DVMT_TIMELINE=1"; run with VMT_LIB=paper_2309_16682_b200/_ab/libvmt_timeline.so).
usage: timeline.py L log2n chunks [prefetch]"""
import ctypes
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2309_16682_b200 as V  # noqa: E402
from paper_2309_16682_b200 import _capi  # noqa: E402

L, lg, chunks = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
pf = int(sys.argv[4]) if len(sys.argv) > 4 else 2
n = 1 << lg
buf = torch.empty(n, dtype=torch.uint32, device="cuda")
g = V.VmtGenerator(5489, V.VmtConfig(L))
g.set_tuning(max_chunks=chunks)
g.set_prefetch(pf)
for _ in range(12):
    g.fill_u32(buf)
torch.cuda.synchronize()
tl = np.zeros(6144, dtype=np.uint64)
lib = ctypes.CDLL(_capi.LIB_PATH)
assert lib.vmt_debug_timeline(tl.ctypes.data_as(ctypes.c_void_p)) == 0
gen = tl[:3072].reshape(1024, 3)
mma = tl[3072:].reshape(1024, 3)
gen = gen[gen[:, 0] > 0]
mma = mma[mma[:, 0] > 0]
t0 = int(min(gen[:, 0].min(), mma[:, 0].min() if len(mma) else gen[:, 0].min()))


def us(a):
    return [round((int(x) - t0) / 1e3, 1) for x in a]


out = {"L": L, "log2n": lg, "chunks": chunks, "prefetch": pf, "gen_ctas": len(gen), "mma_ctas": len(mma),
       "gen_start_us": [min(us(gen[:, 0])), max(us(gen[:, 0]))], "gen_end_us": [min(us(gen[:, 1])), max(us(gen[:, 1]))],
       "gen_sms_distinct": len(set(gen[:, 2].tolist()))}
if len(mma):
    out.update({"mma_start_us": [min(us(mma[:, 0])), max(us(mma[:, 0]))],
                "mma_end_us": [min(us(mma[:, 1])), max(us(mma[:, 1]))],
                "mma_sms_distinct": len(set(mma[:, 2].tolist())),
                "sms_shared": len(set(mma[:, 2].tolist()) & set(gen[:, 2].tolist()))})
    gs = set(gen[:, 2].tolist())
    shared = np.array([s in gs for s in mma[:, 2].tolist()])
    d = (mma[:, 1].astype(np.int64) - mma[:, 0].astype(np.int64)) / 1e3
    out["mma_dur_us_on_gen_sms"] = [round(float(d[shared].min()), 1), round(float(d[shared].max()), 1)] if shared.any() else None
    out["mma_dur_us_on_free_sms"] = [round(float(d[~shared].min()), 1), round(float(d[~shared].max()), 1)] if (~shared).any() else None
    ms = set(mma[:, 2].tolist())
    gshared = np.array([s in ms for s in gen[:, 2].tolist()])
    gd = (gen[:, 1].astype(np.int64) - gen[:, 0].astype(np.int64)) / 1e3
    out["gen_dur_us"] = [round(float(gd.min()), 1), round(float(np.median(gd)), 1), round(float(gd.max()), 1)]
print(json.dumps(out), flush=True)
if len(sys.argv) > 5:
    print("gen", [(int(r[2]), *us(r[:2])) for r in gen][:160])
    print("mma", [(int(r[2]), *us(r[:2])) for r in mma][:160])
