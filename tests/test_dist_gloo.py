"""Multi-rank host logic on CPU (gloo, world size 2): the stream partition
tiles the range, each rank's partial XOR checksum combines (all-gather + fold,
NCCL has no XOR reduction) to the single-rank checksum, and max-over-ranks
timing. The oracle stands in for the per-rank GPU generation here."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, L, q, result_path):
    import sys

    import torch.distributed as dist
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, os.path.join(os.path.dirname(here), "oracle"))
    from oracle import Oracle

    from paper_2309_16682_b200.dist import combine_xor, max_over_ranks, partition
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle()
    lanes = o.dephased_states(5489, L, o.x_pow2_mod(q))
    start, count = partition(total, world, rank)
    part = o.vmt_checksum(lanes, start, count)
    x = combine_xor(part)
    m = max_over_ranks(float(rank + 1))
    with open(f"{result_path}.{rank}", "w") as f:
        f.write(f"{start} {count} {x} {m}")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [3 * 624 * 16 + 17, 1 << 20])
def test_gloo_partition_and_xor_combine(tmp_path, oracle, total):
    world, L, q = 2, 16, 8
    path = str(tmp_path / "res")
    port = _free_port()
    mp.spawn(_worker, args=(world, port, total, L, q, path), nprocs=world, join=True)
    rows = []
    for r in range(world):
        with open(f"{path}.{r}") as f:
            s, c, x, m = f.read().split()
            rows.append((int(s), int(c), int(x), float(m)))
    # partition tiles [0, total) contiguously
    assert rows[0][0] == 0 and rows[0][0] + rows[0][1] == rows[1][0] and rows[1][0] + rows[1][1] == total
    lanes = oracle.dephased_states(5489, L, oracle.x_pow2_mod(q))
    full = oracle.vmt_checksum(lanes, 0, total)
    assert rows[0][2] == rows[1][2] == full
    assert rows[0][3] == rows[1][3] == float(world)


def test_partition_edges():
    from paper_2309_16682_b200.dist import fold_xor, partition
    for total in (0, 1, 7, 1 << 34):
        for world in (1, 2, 3, 8):
            spans = [partition(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and sum(c for _, c in spans) == total
            for (s0, c0), (s1, _) in zip(spans, spans[1:]):
                assert s0 + c0 == s1
    assert fold_xor([1, 3, 0xFFFFFFFF]) == (1 ^ 3 ^ 0xFFFFFFFF)
    with pytest.raises(ValueError):
        partition(10, 2, 2)
