"""GPU parity of the generator batch (config 3) and the single-process
multi-GPU fill (config 4), against the single-generator path (itself pinned
to the reference in test_gpu_parity.py)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2309_16682_b200 as V  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")


def single_streams(seeds, L, q, total):
    out = []
    for s in seeds:
        g = V.VmtEngine(L, int(s), q)
        buf = np.empty(total, np.uint32)
        g.fill_u32(buf)
        out.append(buf)
    return np.stack(out)


@pytest.mark.parametrize("L", [4, 8, 16, 32])
def test_batch_fills_continue_every_stream(L):
    ngen, q = 37, 12
    sizes = [1000, 624 * L + 3, 5, ("skip", 12345), 777, 2 * 624 * L]
    total = sum(s if isinstance(s, int) else s[1] for s in sizes)
    ref = single_streams(range(11, 11 + ngen), L, q, total)
    b = V.VmtBatch(11, ngen, L, q)
    st0 = b.interleaved_states()
    for k, s in enumerate(range(11, 11 + ngen)):
        assert np.array_equal(st0[k], V.VmtEngine(L, s, q).interleaved_state())
    pos = 0
    for s in sizes:
        if not isinstance(s, int):
            b.skip(s[1])
            pos += s[1]
            continue
        dev = torch.empty(ngen * s, dtype=torch.uint32, device="cuda")
        b.fill(dev, s)
        got = dev.cpu().numpy().reshape(ngen, s)
        assert np.array_equal(got, ref[:, pos:pos + s]), (L, s, pos)
        pos += s
        assert b.position == pos
    host = np.empty(ngen * 100, np.uint32)  # host destination
    b.fill(host, 100)
    tail = single_streams(range(11, 11 + ngen), L, q, pos + 100)[:, pos:]
    assert np.array_equal(host.reshape(ngen, 100), tail)


def test_batch_matches_one_shot_config3(golden):
    rows = {r["seed"]: r for r in golden["appendixA"] if r["lanes"] == 16 and r["count"] == 1 << 20}
    n, ngen = 1 << 20, 1024
    b = V.VmtBatch(1, ngen, 16, 16)
    out = torch.empty(n * ngen, dtype=torch.uint32, device="cuda")
    half = n // 2 + 11
    b.fill(out[: half * ngen], half)
    first = out[: half * ngen].view(ngen, half).clone()
    b.fill(out[half * ngen:], n - half)
    rest = out[half * ngen:].view(ngen, n - half)
    v = torch.cat([first, rest], dim=1).cpu().numpy()
    assert int(np.bitwise_xor.reduce(v[0])) == rows[1]["xor"]
    assert int(np.bitwise_xor.reduce(v[1023])) == rows[1024]["xor"]


def test_multi_gpu_fill_partition_and_checksum():
    n = (1 << 24) + 12345
    ref = torch.empty(n, dtype=torch.uint32, device="cuda")
    V.VmtGenerator(5489, V.VmtConfig(32)).fill_u32(ref)
    x_ref = V.VmtGenerator(5489, V.VmtConfig(32)).checksum_xor(n)
    # three parts on distinct devices when the box has them (round robin over
    # the visible GPUs; all on device 0 on a one-GPU box: same partition logic)
    ndev = torch.cuda.device_count()
    devs = [k % ndev for k in range(3)]
    sizes = [n // 3 + (1 if k < n % 3 else 0) for k in range(3)]
    outs = [torch.empty(s, dtype=torch.uint32, device=f"cuda:{d}") for s, d in zip(sizes, devs)]
    x = V.multi_gpu_fill(5489, 32, n, devs, outs)
    torch.cuda.synchronize()
    for d in set(devs):
        torch.cuda.synchronize(d)
    assert torch.equal(torch.cat([o.to(ref.device) for o in outs]), ref)
    assert x == x_ref
    assert V.multi_gpu_fill(5489, 32, n, devs, None) == x_ref  # fused XOR mode


def test_zero_sizes_and_edges():
    """Empty requests are no-ops that leave the stream where it was."""
    g = V.VmtGenerator(5, V.VmtConfig(8, jump_exponent=10))
    ones, bins = g.stat_counts(0)
    assert ones == 0 and int(bins.sum()) == 0 and g.position == 0
    assert g.checksum_xor(0) == 0
    b = V.VmtBatch(1, 3, 8, 10)
    b.fill(np.empty(0, np.uint32), 0)
    assert b.position == 0
    first = V.VmtGenerator(5, V.VmtConfig(8, jump_exponent=10)).next_u32()
    assert g.next_u32() == first
    assert V.multi_gpu_fill(5, 8, 0, [0], None, jump_exponent=10) == 0
