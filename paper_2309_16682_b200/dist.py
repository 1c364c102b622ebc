"""Multi-GPU partitioning of one combined VMT19937 stream.

The stream is a pure function of (seed, lanes, jump exponent, position), so N
ranks split a range [0, total) into contiguous pieces with no data exchange:
rank r owns [floor(r*total/N), floor((r+1)*total/N)) and positions its own
generator there with a jump (``VmtGenerator.skip``). The only collective is the
final combine of per-rank XOR checksums. NCCL has no XOR reduction, so the
4-byte partials are all-gathered and folded locally.
"""
from __future__ import annotations

from typing import Sequence

import torch
import torch.distributed as dist


def partition(total: int, world: int, rank: int) -> tuple[int, int]:
    """(start, count) of rank's contiguous share of [0, total)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    lo = total * rank // world
    hi = total * (rank + 1) // world
    return lo, hi - lo


def fold_xor(parts: Sequence[int]) -> int:
    x = 0
    for p in parts:
        x ^= int(p) & 0xFFFFFFFF
    return x


def collective_device(device: torch.device | str | None = None) -> torch.device:
    """Where the collectives' tensors live: the caller's choice, else this
    rank's current CUDA device under NCCL (which only moves device memory),
    else the CPU (gloo)."""
    if device is not None:
        return torch.device(device)
    if dist.is_initialized() and dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def combine_xor(partial: int, device: torch.device | str | None = None, *, collective: bool = False) -> int:
    """XOR of every rank's 32-bit partial (all-gather + local fold).
    collective=True runs the all-gather even for a single rank (tests)."""
    if not dist.is_initialized() or (dist.get_world_size() == 1 and not collective):
        return partial & 0xFFFFFFFF
    world = dist.get_world_size()
    device = collective_device(device)
    t = torch.tensor([partial & 0xFFFFFFFF], dtype=torch.int64, device=device)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return fold_xor(int(o.item()) for o in out)


def max_over_ranks(value: float, device: torch.device | str | None = None, *, collective: bool = False) -> float:
    """Maximum over ranks (the bench's step time). collective=True runs the
    all-reduce even for a single rank (tests)."""
    if not dist.is_initialized() or (dist.get_world_size() == 1 and not collective):
        return value
    device = collective_device(device)
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
