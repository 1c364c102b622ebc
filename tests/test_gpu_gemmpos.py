"""Steady-state chunk positioning by one int8 tensor-core GEMM (capi_gemmpos.inl):
the chunk states it produces must make every fill word-identical to the
polynomial-jump positioning (itself pinned to the oracle)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2309_16682_b200 as V  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")


def i32(t):
    return t.view(torch.int32)


@pytest.mark.parametrize("L,n,gap", [(32, (1 << 26) + 777, 0), (16, 1 << 27, 0), (32, 1 << 25, 12345), (8, 1 << 28, 0)])
def test_gemm_positioning_matches_polynomial_jumps(L, n, gap):
    ref = V.VmtGenerator(5489, V.VmtConfig(L))
    ref.set_tuning(max_chunks=148)
    ref.set_positioning(1)
    gem = V.VmtGenerator(5489, V.VmtConfig(L))
    gem.set_tuning(max_chunks=148)
    gem.set_positioning(0)
    gem.set_prefetch(0)  # serial GEMM path (the prefetch has its own test)
    a = torch.empty(n, dtype=torch.uint32, device="cuda")
    b = torch.empty(n, dtype=torch.uint32, device="cuda")
    for i in range(6):
        ref.fill_u32(a)
        gem.fill_u32(b)
        torch.cuda.synchronize()
        assert torch.equal(i32(a), i32(b)), (L, n, i)
        ref.skip(gap)
        gem.skip(gap)
    st = gem.positioning_stats()
    assert st["gemm_positionings"] >= 2 and st["cached_matrices"] >= 1
    assert ref.positioning_stats()["gemm_positionings"] == 0


def test_gemm_positioning_mode2_and_shape_changes():
    """Mode 2 uses the GEMM from the second fill; a different fill size or a
    backward seek falls back to the jumps; results stay identical."""
    n = 1 << 25
    ref = V.VmtGenerator(77, V.VmtConfig(32))
    gem = V.VmtGenerator(77, V.VmtConfig(32))
    for g in (ref, gem):
        g.set_tuning(max_chunks=148)
    ref.set_positioning(1)
    gem.set_positioning(2)
    gem.set_prefetch(0)  # serial GEMM path (the prefetch has its own test)
    plan = [n, n, n, n // 2, n, n]
    for i, m in enumerate(plan):
        a = torch.empty(m, dtype=torch.uint32, device="cuda")
        b = torch.empty(m, dtype=torch.uint32, device="cuda")
        if i == 4:
            ref.seek(1000)
            gem.seek(1000)
        ref.fill_u32(a)
        gem.fill_u32(b)
        torch.cuda.synchronize()
        assert torch.equal(i32(a), i32(b)), i
    assert gem.positioning_stats()["gemm_positionings"] >= 2


@pytest.mark.parametrize("L,chunks", [(16, 75), (16, 65), (8, 130)])
def test_small_row_counts_on_own_kernel(L, chunks):
    """Below 2048 lane states (config 1's 75 chunks x 16 lanes = 1200 rows,
    row counts that are not a multiple of the 256-row CTA-pair tile) the
    positioning GEMM is our tcgen05 kernel too (no cuBLAS in the library):
    same words as the polynomial jumps."""
    n = (1 << 25) + 7
    ref = V.VmtGenerator(21, V.VmtConfig(L))
    gem = V.VmtGenerator(21, V.VmtConfig(L))
    for g in (ref, gem):
        g.set_tuning(max_chunks=chunks)
    ref.set_positioning(1)
    gem.set_positioning(2)
    gem.set_prefetch(0)
    a = torch.empty(n, dtype=torch.uint32, device="cuda")
    b = torch.empty(n, dtype=torch.uint32, device="cuda")
    for i in range(4):
        ref.fill_u32(a)
        gem.fill_u32(b)
        torch.cuda.synchronize()
        assert torch.equal(i32(a), i32(b)), i
    assert gem.positioning_stats()["gemm_positionings"] >= 2


def test_single_cta_kernel_matches():
    """The single-CTA tcgen05 form (VMT_POSMMA_SINGLE, M=128 tiles) gives the
    same words as the polynomial jumps."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_2309_16682_b200 as V
n = (1 << 25) + 5
ref = V.VmtGenerator(9, V.VmtConfig(16)); gem = V.VmtGenerator(9, V.VmtConfig(16))
for g in (ref, gem): g.set_tuning(max_chunks=148)
ref.set_positioning(1); gem.set_positioning(2); gem.set_prefetch(0)
a = torch.empty(n, dtype=torch.uint32, device="cuda"); b = torch.empty(n, dtype=torch.uint32, device="cuda")
for i in range(4):
    ref.fill_u32(a); gem.fill_u32(b); torch.cuda.synchronize()
    assert torch.equal(a.view(torch.int32), b.view(torch.int32)), i
assert gem.positioning_stats()["gemm_positionings"] >= 2
print("ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, VMT_POSMMA_SINGLE="1"))
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("tiles,prep,eager", [("1", "1", True), ("2", "2", True), ("1", "2", True), ("2", "1", True),
                                              ("1", "1", False)])
def test_tile_scheduler_and_operand_modes(tiles, prep, eager):
    """The pair kernel's tile order (VMT_POSMMA_TILES: 1 = from the global
    counter, 2 = static round-robin) and the stream its FP4 operand is written
    on (VMT_PREP_AHEAD: 1 = ahead of the generation kernel, 2 = side stream;
    VMT_NO_EAGER_FP4: not right behind the previous prefetch) never change a word: co-resident prefetch with fewer chunks than SMs, one
    chunk per SM, ragged fill sizes and a serial GEMM, against the polynomial
    jumps."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_2309_16682_b200 as V
for L, n, chunks in ((16, (1 << 25) + 4097, 60), (16, 1 << 26, 148), (32, (1 << 26) + 33, 37), (8, 1 << 26, 100)):
    ref = V.VmtGenerator(11, V.VmtConfig(L)); pre = V.VmtGenerator(11, V.VmtConfig(L)); ser = V.VmtGenerator(11, V.VmtConfig(L))
    for g in (ref, pre, ser): g.set_tuning(max_chunks=chunks)
    ref.set_positioning(1); ref.set_prefetch(0)
    pre.set_prefetch(2)
    ser.set_positioning(2); ser.set_prefetch(0)
    a = torch.empty(n, dtype=torch.uint32, device="cuda"); b = torch.empty_like(a); c = torch.empty_like(a)
    for i in range(7):
        ref.fill_u32(a); pre.fill_u32(b); ser.fill_u32(c); torch.cuda.synchronize()
        assert torch.equal(a.view(torch.int32), b.view(torch.int32)), (L, chunks, i, "prefetch")
        assert torch.equal(a.view(torch.int32), c.view(torch.int32)), (L, chunks, i, "serial")
    assert pre.prefetch_stats()["used"] >= 3, (L, chunks, pre.prefetch_stats())
    assert ser.positioning_stats()["gemm_positionings"] >= 3
print("ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, VMT_POSMMA_TILES=tiles, VMT_PREP_AHEAD=prep,
                                **({} if eager else {"VMT_NO_EAGER_FP4": "1"})))
    assert r.returncode == 0 and "ok" in r.stdout, (r.stdout[-500:], r.stderr[-2000:])


def test_gemm_positioning_in_fused_modes():
    """The fused consumers (XOR checksum, statistics) and the float fills go
    through the same positioning: repeated calls agree with the jump path."""
    n = (1 << 26) + 3
    ref = V.VmtGenerator(3, V.VmtConfig(32))
    gem = V.VmtGenerator(3, V.VmtConfig(32))
    for g in (ref, gem):
        g.set_tuning(max_chunks=148)
    ref.set_positioning(1)
    gem.set_positioning(2)
    gem.set_prefetch(0)  # serial GEMM path (the prefetch has its own test)
    for _ in range(3):
        assert ref.checksum_xor(n) == gem.checksum_xor(n)
    for _ in range(3):
        o1, b1 = ref.stat_counts(n)
        o2, b2 = gem.stat_counts(n)
        assert o1 == o2 and np.array_equal(b1, b2)
    f1 = torch.empty(n, dtype=torch.float32, device="cuda")
    f2 = torch.empty(n, dtype=torch.float32, device="cuda")
    for _ in range(3):
        ref.fill_f32(f1)
        gem.fill_f32(f2)
        torch.cuda.synchronize()
        assert torch.equal(f1.view(torch.int32), f2.view(torch.int32))
    assert gem.positioning_stats()["gemm_positionings"] >= 6


def test_gemm_positioning_reuses_matrix_with_block_advance():
    """Three fill sizes cycling (block deltas D, D+1, D+2): the deltas above
    a cached one reuse its matrix and regenerate the remaining blocks in place
    (vmt_advance_blocks_kernel); words stay identical."""
    bw = 624 * 32
    ref = V.VmtGenerator(11, V.VmtConfig(32))
    gem = V.VmtGenerator(11, V.VmtConfig(32))
    for g in (ref, gem):
        g.set_tuning(max_chunks=148)
    ref.set_positioning(1)
    gem.set_positioning(2)
    gem.set_prefetch(0)  # serial GEMM path (the prefetch has its own test)
    for k in range(10):
        n = bw * (3000 + (k % 3))
        a = torch.empty(n, dtype=torch.uint32, device="cuda")
        b = torch.empty(n, dtype=torch.uint32, device="cuda")
        ref.fill_u32(a)
        gem.fill_u32(b)
        torch.cuda.synchronize()
        assert torch.equal(i32(a), i32(b)), k
    st = gem.positioning_stats()
    assert 1 <= st["cached_matrices"] <= 2 and st["gemm_positionings"] >= 7


def test_gemm_positioned_stream_pinned_to_oracle(golden):
    """The bench range [0, 2^34) produced in four consecutive 2^32-word calls
    with GEMM positioning from the second call on: the XOR of all words (fused
    checksums, and the stored words) equals the C oracle's pinned value."""
    from test_gpu_parity import xor_reduce_inplace
    c = golden["c4_full"]
    g = V.VmtGenerator(c["seed"], V.VmtConfig(c["lanes"]))
    g.set_positioning(2)
    g.set_prefetch(0)  # serial GEMM path (the prefetch has its own test)
    x = 0
    for _ in range(4):
        x ^= g.checksum_xor(1 << 32)
    assert x == c["xor"] and g.positioning_stats()["gemm_positionings"] >= 2
    g = V.VmtGenerator(c["seed"], V.VmtConfig(c["lanes"]))
    g.set_positioning(2)
    g.set_prefetch(0)  # serial GEMM path (the prefetch has its own test)
    out = torch.empty(c["count"], dtype=torch.uint32, device="cuda")
    for k in range(4):
        g.fill_u32(out[k << 32:(k + 1) << 32])
    assert g.positioning_stats()["gemm_positionings"] >= 3
    assert xor_reduce_inplace(out) == c["xor"]


@pytest.mark.parametrize("L,n,gap", [(32, (1 << 26) + 777, 0), (32, 1 << 27, 4321), (16, 1 << 27, 0),
                                     (32, 1 << 32, 0)])
def test_tensor_core_prefetch_matches_polynomial_jumps(L, n, gap, chunks=148):
    """VMT_PREFETCH_TENSOR: the next fill's chunk states come from the
    hand-written tcgen05 kernel (vmt_posmma.cuh) running beside the generation
    kernel; every fill must equal the jump-positioned reference."""
    ref = V.VmtGenerator(4242, V.VmtConfig(L))
    ref.set_tuning(max_chunks=chunks)
    ref.set_positioning(1)
    ref.set_prefetch(0)
    tc = V.VmtGenerator(4242, V.VmtConfig(L))
    tc.set_tuning(max_chunks=chunks)
    tc.set_prefetch(2)
    a = torch.empty(n, dtype=torch.uint32, device="cuda")
    b = torch.empty(n, dtype=torch.uint32, device="cuda")
    for i in range(8):
        ref.fill_u32(a)
        tc.fill_u32(b)
        torch.cuda.synchronize()
        assert torch.equal(i32(a), i32(b)), (L, n, i)
        ref.skip(gap)
        tc.skip(gap)
    st = tc.prefetch_stats()
    if L == 32:  # the 32-lane store kernel leaves room for the GEMM CTA
        # (2^32 words = 215092.5 blocks: the block delta alternates, one
        # cached matrix + in-place regeneration serves both)
        assert st["tensor_prefetches"] >= 4 and st["used"] >= 4, st
    # a different size next: the prefetched states are discarded, words stay exact
    m = n // 3
    a2 = torch.empty(m, dtype=torch.uint32, device="cuda")
    b2 = torch.empty(m, dtype=torch.uint32, device="cuda")
    ref.fill_u32(a2)
    tc.fill_u32(b2)
    torch.cuda.synchronize()
    assert torch.equal(i32(a2), i32(b2))


def test_tensor_core_prefetch_host_destination_and_streams():
    """The prefetch in the host-destination path (1 GiB staged segments) and
    with the caller switching CUDA streams between fills: identical words."""
    n = (1 << 28) * 3 + 1234  # three full segments + a ragged one
    ref = V.VmtGenerator(99, V.VmtConfig(32))
    ref.set_positioning(1)
    ref.set_prefetch(0)
    tc = V.VmtGenerator(99, V.VmtConfig(32))
    tc.set_prefetch(2)
    a = torch.empty(n, dtype=torch.uint32, pin_memory=True)
    b = torch.empty(n, dtype=torch.uint32, pin_memory=True)
    ref.fill_u32(a)
    tc.fill_u32(b)
    assert torch.equal(i32(a), i32(b))
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    m = 1 << 27
    da = torch.empty(m, dtype=torch.uint32, device="cuda")
    db = torch.empty(m, dtype=torch.uint32, device="cuda")
    for i in range(8):
        s = streams[i % 2]
        ref.fill_u32(da)
        tc.fill_u32(db, stream=s.cuda_stream)
        torch.cuda.synchronize()
        assert torch.equal(i32(da), i32(db)), i
    assert tc.prefetch_stats()["used"] >= 2, tc.prefetch_stats()


def test_tensor_core_prefetch_padded_rows():
    """99 chunks x 32 lanes = 3168 lane states: the last 128-row tile of the
    tcgen05 GEMM is padded with zero rows whose results are not stored."""
    test_tensor_core_prefetch_matches_polynomial_jumps(32, (1 << 27) + 99, 0, chunks=99)


def test_tensor_core_prefetch_two_ctas_per_sm_f32():
    """Config 2's shape: L=8, 2^28 float32 per fill, 296 chunks = two
    generation CTAs per SM plus the co-resident positioning CTA."""
    n = 1 << 28
    ref = V.VmtGenerator(42, V.VmtConfig(8))
    ref.set_positioning(1)
    ref.set_prefetch(0)
    tc = V.VmtGenerator(42, V.VmtConfig(8))
    tc.set_prefetch(2)
    a = torch.empty(n, dtype=torch.float32, device="cuda")
    b = torch.empty(n, dtype=torch.float32, device="cuda")
    for i in range(8):
        ref.fill_f32(a)
        tc.fill_f32(b)
        torch.cuda.synchronize()
        assert torch.equal(a.view(torch.int32), b.view(torch.int32)), i
    st = tc.prefetch_stats()
    assert st["tensor_prefetches"] >= 3 and st["used"] >= 3, st


def test_tensor_core_prefetch_two_generators_interleaved():
    """Two handles with prefetches in flight at the same time (each on its own
    side stream), fills interleaved, one destroyed mid-way: every word equals
    its jump-positioned reference."""
    n = (1 << 27) + 4321
    refs = [V.VmtGenerator(s, V.VmtConfig(32)) for s in (11, 12)]
    tcs = [V.VmtGenerator(s, V.VmtConfig(32)) for s in (11, 12)]
    for r in refs:
        r.set_tuning(max_chunks=148)
        r.set_positioning(1)
        r.set_prefetch(0)
    for t in tcs:
        t.set_tuning(max_chunks=148)
        t.set_prefetch(2)
    a = torch.empty(n, dtype=torch.uint32, device="cuda")
    b = torch.empty(n, dtype=torch.uint32, device="cuda")
    for i in range(7):
        for k in range(len(tcs)):
            refs[k].fill_u32(a)
            tcs[k].fill_u32(b)
            torch.cuda.synchronize()
            assert torch.equal(i32(a), i32(b)), (i, k)
        if i == 4:
            del tcs[1], refs[1]  # destroyed with its prefetch possibly in flight
    assert tcs[0].prefetch_stats()["used"] >= 3


@pytest.mark.parametrize("L,chunks,n", [(16, 20, (1 << 24) + 33), (32, 9, 1 << 24), (16, 50, 1 << 26)])
@pytest.mark.parametrize("prefetch", [0, 2])
def test_gemm_positioning_small_row_counts(L, chunks, n, prefetch):
    """The GEMM positions from 256 lane states since round 2 (320, 288 and 800
    rows here, one to four pair tiles): serial and co-resident, every fill
    word-identical to the polynomial-jump positioning."""
    ref = V.VmtGenerator(99, V.VmtConfig(L))
    ref.set_tuning(max_chunks=chunks)
    ref.set_positioning(1)
    ref.set_prefetch(0)
    gem = V.VmtGenerator(99, V.VmtConfig(L))
    gem.set_tuning(max_chunks=chunks)
    gem.set_prefetch(prefetch)
    a = torch.empty(n, dtype=torch.uint32, device="cuda")
    b = torch.empty(n, dtype=torch.uint32, device="cuda")
    for i in range(7):
        ref.fill_u32(a)
        gem.fill_u32(b)
        torch.cuda.synchronize()
        assert torch.equal(i32(a), i32(b)), (L, chunks, n, prefetch, i)
    assert gem.positioning_stats()["cached_matrices"] >= 1
    if prefetch:
        assert gem.prefetch_stats()["used"] >= 2
    else:
        assert gem.positioning_stats()["gemm_positionings"] >= 2


@pytest.mark.parametrize("L,chunks,n", [(1, 300, (1 << 22) + 5), (2, 296, (1 << 23) + 77), (4, 148, (1 << 24) + 1),
                                         (8, 296, (1 << 25) + 4097)])
def test_gemm_positioning_and_block_advance_at_small_lane_counts(L, chunks, n):
    """GEMM positioning with the in-place block advance (fill sizes that are
    not a multiple of the block: every repeat regenerates one or two blocks
    after the GEMM) at 1, 2, 4 and 8 lanes -- the advance kernel's scalar
    (L < 4) and 16-byte paths -- against the polynomial jumps."""
    ref = V.VmtGenerator(1234, V.VmtConfig(L))
    gem = V.VmtGenerator(1234, V.VmtConfig(L))
    for g in (ref, gem):
        g.set_tuning(max_chunks=chunks)
        g.set_prefetch(0)
    ref.set_positioning(1)
    gem.set_positioning(2)
    a = torch.empty(n, dtype=torch.uint32, device="cuda")
    b = torch.empty(n, dtype=torch.uint32, device="cuda")
    for i in range(8):
        ref.fill_u32(a)
        gem.fill_u32(b)
        torch.cuda.synchronize()
        assert torch.equal(i32(a), i32(b)), (L, chunks, n, i)
    assert gem.positioning_stats()["gemm_positionings"] >= 3, gem.positioning_stats()


def test_randomised_positioning_stress():
    """profiles/scripts/stress_positioning.py: 150 random fills over four
    generators (L = 32/16/8/16) with shape changes, skips and chunk-count
    changes between them -- prefetched, serial-GEMM and jump-positioned fills in
    whatever order they fall -- every fill identical to jump positioning."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "profiles", "scripts", "stress_positioning.py"), "150", "4"],
                       cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.startswith("ok"), (r.stdout[-500:], r.stderr[-2000:])
