"""The NCCL side of the multi-GPU path on one B200 (the pool gives one GPU
per call, so this is a single-rank communicator): process-group set-up with
the bench's device binding, and the collectives dist.py issues -- the
checksum all-gather, the step-time max all-reduce, the per-rank record
all_gather_object -- on CUDA tensors through NCCL. The partition / fold logic
for N > 1 is covered with gloo on CPU (test_dist_gloo.py)."""
import os

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import torch.distributed as dist  # noqa: E402

from paper_2309_16682_b200.dist import collective_device, combine_xor, max_over_ranks  # noqa: E402


@pytest.fixture(scope="module")
def nccl_group():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    if not dist.is_nccl_available():
        pytest.fail("torch has no NCCL backend")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29571")
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    yield dev
    dist.destroy_process_group()


def test_nccl_collectives_of_the_bench(nccl_group):
    dev = nccl_group
    assert dist.get_backend() == "nccl"
    assert collective_device() == dev
    assert combine_xor(0x1234ABCD, collective=True) == 0x1234ABCD
    assert combine_xor(0x1234ABCD) == 0x1234ABCD
    assert max_over_ranks(12.5, collective=True) == 12.5
    rec = [None]
    dist.all_gather_object(rec, {"rank": 0, "ms": 12.5})
    assert rec == [{"rank": 0, "ms": 12.5}]
    ok = torch.tensor([1], device=dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    assert int(ok.item()) == 1
    dist.barrier()
