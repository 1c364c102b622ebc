"""Pinned D2H copy throughput with 1, 2 and 4 concurrent streams (the e2e
fill's link): 16 GiB moved as 1 GiB or 256 MiB pieces."""
import json
import time

import torch

dev = torch.device("cuda", 0)
total = 16 << 30
src = torch.empty(1 << 28, dtype=torch.uint32, device=dev)  # 1 GiB
src.fill_(7)
dst = torch.empty(total // 4, dtype=torch.uint32, pin_memory=True)
for piece in (1 << 30, 1 << 28):
    for ns in (1, 2, 4):
        streams = [torch.cuda.Stream(dev) for _ in range(ns)]
        words = piece // 4
        n = total // piece
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i in range(n):
                s = streams[i % ns]
                with torch.cuda.stream(s):
                    dst[i * words:(i + 1) * words].copy_(src[:words], non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        print(json.dumps({"piece_mib": piece >> 20, "streams": ns, "gbs": round(total / dt / 1e9, 2)}), flush=True)
