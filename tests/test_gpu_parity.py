"""GPU parity: the sm_100a kernels, called through the C ABI, against the
reference's golden vectors and the C oracle. Bit-exact everywhere (integer
and exactly-rounded conversions)."""
import hashlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2309_16682_b200 as V  # noqa: E402
from conftest import dephase_poly, oracle_window  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def dev_u32(n):
    return torch.empty(n, dtype=torch.uint32, device="cuda")


def host(t):
    return t.cpu().numpy()


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")


def test_appendix_a_l16_q16(golden):
    row = [r for r in golden["appendixA"] if r["lanes"] == 16 and r["seed"] == 5489][0]
    g = V.VmtEngine(16, 5489, 16)
    out = dev_u32(row["count"])
    g.fill_u32(out)
    torch.cuda.synchronize()
    v = host(out)
    assert list(v[:4]) == row["first4"] and int(v[-1]) == row["last"]
    assert int(np.bitwise_xor.reduce(v)) == row["xor"] == 0x5E141D5B


@pytest.mark.parametrize("q", [6, 8, 16])
@pytest.mark.parametrize("L", [1, 2, 4, 8, 16])
def test_engine_streams(golden, gnpz, L, q):
    streams = gnpz("engine_streams.npz")
    for e in golden["engine"]:
        if e["lanes"] != L or e["q"] != q:
            continue
        g = V.VmtEngine(L, e["seed"], q)
        out = dev_u32(e["count"])
        g.fill_u32(out)
        v = host(out)
        assert np.array_equal(v[:4096], streams[f"L{L}_q{q}_s{e['seed']}"])
        assert sha(v) == e["sha"]


def test_query_modes_identical():
    # test_engine.cpp:81-109 / acceptance.cpp:109-135 (n = 100000)
    n = 100000
    a = V.VmtEngine(4, 5489, 8)
    b = V.VmtEngine(4, 5489, 8)
    c = V.VmtEngine(4, 5489, 8)
    d = V.VmtEngine(4, 5489, 8)
    va = np.array([a.next_u32() for _ in range(n)], np.uint32)
    vb = np.concatenate([b.next_block16() for _ in range((n + 15) // 16)])[:n]
    vc = np.concatenate([c.next_block_state() for _ in range(-(-n // 2496))])[:n]
    vd = np.empty(n, np.uint32)
    pos = 0
    for k in (1, 15, 16, 2496, 3, 7777, 10):  # ragged bulk fills, host destination
        d.fill_u32(vd[pos:pos + k])
        pos += k
    d.fill_u32(vd[pos:])
    assert np.array_equal(va, vb) and np.array_equal(va, vc) and np.array_equal(va, vd)


def test_mid_buffer_block16_and_cadence():
    mixed = V.VmtEngine(4, 42, 6)
    plain = V.VmtEngine(4, 42, 6)
    for prefix in (1, 2, 3):
        for _ in range(prefix):
            assert mixed.next_u32() == plain.next_u32()
        buf = mixed.next_block16()
        assert list(buf) == [plain.next_u32() for _ in range(16)]
    g = V.VmtEngine(4, 7, 6)
    g.next_block_state()
    g.next_u32()
    with pytest.raises(V.LogicError):
        g.next_block_state()


def test_interleaved_state_after_three_blocks(gnpz):
    g = V.VmtEngine(4, 31337, 10)
    for _ in range(3):
        g.next_block_state()
    assert np.array_equal(g.interleaved_state(), gnpz("engine_state_L4_q10_s31337_b3.npy"))


def test_dephased_state_export(gnpz):
    ref = gnpz("ref_jumps.npz")["dephased_L32_q16_s5489"]
    g = V.VmtEngine(32, 5489, 16)
    assert np.array_equal(g.interleaved_state().reshape(624, 32).T, ref)
    ref16 = gnpz("ref_jumps.npz")["dephased_L16_q16_s1"]
    g = V.VmtEngine(16, 1, 16)
    assert np.array_equal(g.interleaved_state().reshape(624, 16).T, ref16)


def test_config4_windows_q16_via_skip(golden):
    for w in golden["c4_windows_q16"]:
        g = V.VmtEngine(32, 5489, 16)
        g.skip(w["start_word"])
        out = dev_u32(w["count"])
        g.fill_u32(out)
        v = host(out)
        assert list(v[:8]) == w["head"] and sha(v) == w["sha"]


@pytest.mark.parametrize("L", [8, 16, 32])
def test_full_period_default_jump(oracle, full_polys, L):
    """Library default de-phasing (q = 19937 - log2 L) vs the oracle's
    polynomial de-phasing (parity pinned transitively)."""
    q = 19937 - (L.bit_length() - 1)
    lanes = oracle.dephased_states(5489, L, full_polys[f"q{q}"])
    g = V.VmtGenerator(5489, V.VmtConfig(L))
    assert g.jump_exponent() == q
    assert np.array_equal(g.interleaved_state().reshape(624, L).T, lanes)
    n = 1 << 20
    out = dev_u32(n)
    g.fill_u32(out)
    v = host(out)
    assert np.array_equal(v, oracle.vmt_stream(lanes, 0, n))
    assert int(v[0]) == 3499211612  # output[0] is the scalar first output for seed 5489


@pytest.mark.parametrize("max_chunks", [1, 7, 0])
def test_chunked_fill_appendix_a_l8(golden, max_chunks):
    row = [r for r in golden["appendixA"] if r["lanes"] == 8][0]  # 2^28 words
    g = V.VmtEngine(8, 42, 16)
    g.set_tuning(max_chunks=max_chunks)
    out = dev_u32(row["count"])
    g.fill_u32(out)
    v = host(out)
    assert int(np.bitwise_xor.reduce(v)) == row["xor"] == 0x3837517C
    assert list(v[:4]) == row["first4"] and int(v[-1]) == row["last"]


def test_xor_checksum_matches_store(golden):
    row = [r for r in golden["appendixA"] if r["lanes"] == 16 and r["seed"] == 5489][0]
    g = V.VmtEngine(16, 5489, 16)
    assert g.checksum_xor(row["count"]) == row["xor"]
    # continuation: xor of the next window equals the stored next window
    a = V.VmtEngine(16, 5489, 16)
    a.skip(row["count"])
    out = dev_u32(12345)
    a.fill_u32(out)
    assert g.checksum_xor(12345) == int(np.bitwise_xor.reduce(host(out)))


@pytest.mark.parametrize("L", [8, 16, 32])
def test_ragged_positions(oracle, L):
    q = 8
    lanes = oracle.dephased_states(99, L, oracle.x_pow2_mod(q))
    total = 3 * 624 * L + 1001
    ref = oracle.vmt_stream(lanes, 0, total)
    g = V.VmtEngine(L, 99, q)
    got = []
    for k in (0, 1, 2, 3, 5, 624 * L - 11, 4, 624 * L + 1, 7, 1000):
        t = dev_u32(max(k, 1))
        g.fill_u32(t, k)
        got.append(host(t)[:k])
    rest = total - sum(len(x) for x in got)
    t = dev_u32(rest)
    g.fill_u32(t)
    got.append(host(t))
    assert np.array_equal(np.concatenate(got), ref)


def test_float_conversions(oracle):
    L, q, n = 8, 16, (1 << 20) + 6
    lanes = oracle.dephased_states(42, L, oracle.x_pow2_mod(q))
    u = oracle.vmt_stream(lanes, 0, 2 * n)
    f32 = ((u[:n] >> 8).astype(np.float32) * np.float32(2.0 ** -24))
    f64 = u[:n].astype(np.float64) * 2.0 ** -32
    r3 = (u[:n].astype(np.float64) + 0.5) * 2.0 ** -32
    a, b = u[0:2 * n:2], u[1:2 * n:2]
    r53 = ((a >> 5).astype(np.float64) * 67108864.0 + (b >> 6).astype(np.float64)) * 2.0 ** -53
    g = V.VmtEngine(L, 42, q)
    t = torch.empty(n, dtype=torch.float32, device="cuda")
    g.fill_f32(t)
    assert np.array_equal(host(t).view(np.uint32), f32.view(np.uint32))
    assert host(t).max() < 1.0
    for rule, ref in ((V.VMT_F64_32, f64), (V.VMT_F64_REAL3, r3), (V.VMT_F64_RES53, r53)):
        g = V.VmtEngine(L, 42, q)
        t = torch.empty(n, dtype=torch.float64, device="cuda")
        g.fill_f64(t, rule=rule)
        assert np.array_equal(host(t).view(np.uint64), ref.view(np.uint64)), rule


def test_batch_generators(golden, oracle):
    rows = {r["seed"]: r for r in golden["appendixA"] if r["lanes"] == 16 and r["count"] == 1 << 20}
    n, ngen = 1 << 20, 1024
    out = dev_u32(n * ngen)
    V.batch_fill_u32(out, 1, ngen, 16, n, jump_exponent=16)
    v = host(out).reshape(ngen, n)
    assert int(np.bitwise_xor.reduce(v[0])) == rows[1]["xor"] == 0xA63A3C52
    assert int(np.bitwise_xor.reduce(v[1023])) == rows[1024]["xor"] == 0xD18F46A1
    poly = oracle.x_pow2_mod(16)
    for gi in (5, 511, 777):
        lanes = oracle.dephased_states(gi + 1, 16, poly)
        assert np.array_equal(v[gi, :20000], oracle.vmt_stream(lanes, 0, 20000))


def test_jump_states_config5(gnpz, oracle):
    c5 = gnpz("c5_ref.npz")
    seeds = np.arange(1, 4097, dtype=np.uint32)
    st = V.seed_states(seeds)
    assert np.array_equal(st[0], oracle.seed_words(1))
    d = oracle.mt64(7, 4096)
    out = V.jump_states(st, d)
    for i in range(8):
        assert np.array_equal(oracle.mt_stream_from_words(out[i], 624), c5[f"s{i + 1}"]), i
    for i in (100, 2047, 4095):
        j = oracle.poly_jump(st[i], oracle.x_pow_mod(int(d[i])))
        assert np.array_equal(out[i], j)


def test_jump_states_small_and_edge_distances(oracle):
    """Distances whose low 16 bits are applied by direct advance
    (vmt_advance_steps_kernel) and whose high bits by table jumps: every
    state word equals the oracle's polynomial jump, word 0 included."""
    seeds = np.arange(11, 11 + 12, dtype=np.uint32)
    st = V.seed_states(seeds)
    d = np.array([0, 1, 226, 227, 623, 624, 625, 65535, 65536, 65537, (1 << 40) + 12345, (1 << 64) - 1],
                 dtype=np.uint64)
    out = V.jump_states(st, d)
    for i in range(len(d)):
        j = oracle.poly_jump(st[i], oracle.x_pow_mod(int(d[i])))
        assert np.array_equal(out[i], j), int(d[i])


def test_create_from_states_roundtrip(oracle):
    lanes = oracle.dephased_states(7, 8, oracle.x_pow2_mod(12))
    g = V.VmtGenerator(0, lane_states=lanes)
    out = dev_u32(50000)
    g.fill_u32(out)
    assert np.array_equal(host(out), oracle.vmt_stream(lanes, 0, 50000))


def test_empty_fill_and_host_destination():
    g = V.VmtEngine(16, 5489, 16)
    g.fill_u32(dev_u32(1), 0)
    h = np.empty(10000, np.uint32)
    g.fill_u32(h)
    r = V.VmtEngine(16, 5489, 16)
    d = dev_u32(10000)
    r.fill_u32(d)
    assert np.array_equal(h, host(d))


@pytest.mark.parametrize("L,variants", [(32, [1, 3, 4, 6, 7, 8]), (16, [1, 3, 4, 5, 6, 7]), (8, [1, 3, 4, 5]), (4, [4, 5]),
                                        (2, [4, 5]), (1, [5])])
def test_kernel_variants_identical(oracle, L, variants):
    """Every CTA-shape variant (run length, vector width, window, TMA bulk
    stores) emits the same words, across chunk boundaries and ragged ends."""
    q = 10
    lanes = oracle.dephased_states(2024, L, oracle.x_pow2_mod(q)) if L > 1 else oracle.seed_words(2024)[None]
    start, n = 3 * 624 * L + 5, 40 * 624 * L + 77
    ref = oracle.vmt_stream(lanes, start, n)
    for v in variants:
        for chunks in (1, 5):
            g = V.VmtEngine(L, 2024, q)
            g.set_tuning(max_chunks=chunks, variant=v)
            g.skip(start)
            out = dev_u32(n + 8)[4:4 + n]  # 16-byte misaligned destination too
            g.fill_u32(out)
            assert np.array_equal(host(out), ref), (L, v, chunks)
            g2 = V.VmtEngine(L, 2024, q)
            g2.set_tuning(max_chunks=chunks, variant=v)
            g2.skip(start)
            out2 = dev_u32(n)
            g2.fill_u32(out2)
            assert np.array_equal(host(out2), ref), (L, v, chunks, "aligned")
            x = V.VmtEngine(L, 2024, q)
            x.set_tuning(max_chunks=chunks, variant=v)
            x.skip(start)
            assert x.checksum_xor(n) == int(np.bitwise_xor.reduce(ref)), (L, v, chunks, "xor")


def test_prefetched_positioning_matches(oracle):
    """Consecutive large fills reuse chunk states prefetched during the
    previous fill (same size, same gap); mispredictions fall back. The words
    must be identical to the oracle either way."""
    L, q = 16, 8
    lanes = oracle.dephased_states(77, L, oracle.x_pow2_mod(q))
    n, gap = (1 << 24) + 3, 12345
    plan = [(n, 0), (n, 0), (n, gap), (n, gap), (n - 7, 0), (n, 0)]
    pos = 0
    g = V.VmtEngine(L, 77, q)
    g.set_prefetch(True)
    for i, (size, skip) in enumerate(plan):
        g.skip(skip)
        pos += skip
        out = dev_u32(size)
        g.fill_u32(out)
        v = host(out)
        assert int(np.bitwise_xor.reduce(v)) == oracle.vmt_checksum(lanes, pos, size), i
        assert np.array_equal(v[:1000], oracle.vmt_stream(lanes, pos, 1000)), i
        pos += size
    st = g.stats()
    assert st["jump_launches"] >= 3


def test_float_conversions_tma_variant(oracle):
    L, q, n = 16, 12, 300000
    lanes = oracle.dephased_states(42, L, oracle.x_pow2_mod(q))
    u = oracle.vmt_stream(lanes, 0, n)
    g = V.VmtEngine(L, 42, q)
    g.set_tuning(variant=6)
    t = torch.empty(n, dtype=torch.float32, device="cuda")
    g.fill_f32(t)
    assert np.array_equal(host(t), (u >> 8).astype(np.float32) * np.float32(2.0 ** -24))
    g = V.VmtEngine(L, 42, q)
    g.set_tuning(variant=6)
    t = torch.empty(n, dtype=torch.float64, device="cuda")
    g.fill_f64(t)
    assert np.array_equal(host(t), u.astype(np.float64) * 2.0 ** -32)


def test_profiling_events_cover_every_fill():
    """vmt_set_profiling / vmt_last_timings / vmt_profile_totals: one event
    triplet per fill, summed over all fills (bench.py's kernel breakdown)."""
    g = V.VmtEngine(16, 3, 10)
    out = dev_u32(1 << 22)
    with pytest.raises(V.LogicError):
        g.last_timings()
    g.set_profiling(True)
    for _ in range(5):
        g.fill_u32(out)
    j, gm = g.last_timings()
    assert gm > 0 and j >= 0
    n, jt, gt = g.profile_totals()
    assert n == 5 and gt >= gm and jt >= 0
    assert g.profile_totals() == (0, 0.0, 0.0)
    g.set_profiling(False)
    g.fill_u32(out)
    assert g.profile_totals()[0] == 0


def xor_reduce_inplace(t):
    """XOR of all words of a 1-D uint32 CUDA tensor, by in-place halving."""
    t = t.view(torch.int32)  # (bitwise ops on uint32 are not implemented for CUDA)
    n = t.numel()
    while n > 1:
        h = n // 2
        torch.bitwise_xor(t[:h], t[n - h:n], out=t[:h])  # an odd middle word stays at t[h]
        n = n - h
    return int(t[0].item()) & 0xFFFFFFFF


# Window offsets into the config-4 stream [0, 2^34): three drawn from a fixed
# seed, plus windows straddling the rank boundaries of the N=8, 4 and 2 splits
# (2^31, 2^32, 2^33) and the last 2^20 words (BASELINE.json configs[3]:
# "2^20-word windows at random offsets against the CPU oracle").
C4_WIN = 1 << 20
C4_OFFSETS = sorted([int(v) for v in np.random.default_rng(2309).integers(0, (1 << 34) - C4_WIN, 3)]
                    + [(1 << 31) - (C4_WIN >> 1), (1 << 32) - 12345, (1 << 33) - (C4_WIN >> 1) + 7,
                       3 * (1 << 32) - 99, (1 << 34) - C4_WIN])


@pytest.fixture(scope="module")
def c4_oracle_windows(oracle, full_polys):
    lanes = oracle.dephased_states(5489, 32, full_polys["q19932"])
    return {s: oracle_window(oracle, 5489, 32, None, s, C4_WIN, dephased=lanes) for s in C4_OFFSETS}


def test_bench_workload_pinned_to_oracle(golden, c4_oracle_windows):
    """The bench's config-4 step itself (L=32, seed 5489, full period, words
    [0, 2^34), 64 GiB), stored in HBM in one call: the C oracle's XOR of every
    word (tests/golden, make_golden.py c4_full) equals both the fused checksum
    and the XOR of the 64 GiB actually stored; 2^20-word windows of the stored
    buffer at random offsets and across the N=2/4/8 rank boundaries equal the
    C oracle word for word (windows: proj/tests/test_engine.cpp:37-49,
    acceptance.cpp:222-232)."""
    c = golden["c4_full"]
    n = c["count"]
    g = V.VmtGenerator(c["seed"], V.VmtConfig(c["lanes"]))
    assert g.jump_exponent() == c["q"]
    assert g.checksum_xor(n) == c["xor"]
    out = dev_u32(n)
    V.VmtGenerator(c["seed"], V.VmtConfig(c["lanes"])).fill_u32(out)
    for start, ref in c4_oracle_windows.items():
        assert np.array_equal(host(out[start:start + C4_WIN]), ref), start
    assert xor_reduce_inplace(out) == c["xor"]
    del out


@pytest.mark.parametrize("start", C4_OFFSETS)
def test_config4_full_period_windows_vs_oracle(c4_oracle_windows, start):
    """Each window again through a generator positioned with skip() -- the way
    a rank of the N-GPU split positions itself -- in store mode and in the
    fused-XOR (no-store) mode, against the C oracle at q=19932."""
    ref = c4_oracle_windows[start]
    g = V.VmtGenerator(5489, V.VmtConfig(32))
    g.skip(start)
    w = dev_u32(C4_WIN)
    g.fill_u32(w)
    assert np.array_equal(host(w), ref), start
    h = V.VmtGenerator(5489, V.VmtConfig(32))
    h.skip(start)
    assert h.checksum_xor(C4_WIN) == int(np.bitwise_xor.reduce(ref)), start
    # the fused path continues exactly where the window ends
    nxt = dev_u32(1000)
    g.fill_u32(nxt)
    assert h.checksum_xor(1000) == int(np.bitwise_xor.reduce(host(nxt)))


def test_config1_full_size_vs_oracle(oracle, full_polys):
    """c1 as BASELINE.json states it: L=16, seed 5489, default (full-period)
    de-phasing, 2^26 words, every word against the oracle."""
    n = 1 << 26
    lanes = oracle.dephased_states(5489, 16, full_polys["q19933"])
    ref = oracle.vmt_stream(lanes, 0, n)
    g = V.VmtGenerator(5489, V.VmtConfig(16))
    out = dev_u32(n)
    g.fill_u32(out)
    assert np.array_equal(host(out), ref)


def test_config2_full_size_vs_oracle(oracle, full_polys):
    """c2 as BASELINE.json states it: L=8, seed 42, default de-phasing, 2^28
    values as float32 and as float64 (both conversions of the same words),
    every value bit-exact against the documented rules on the oracle stream."""
    n = 1 << 28
    lanes = oracle.dephased_states(42, 8, full_polys["q19934"])
    u = oracle.vmt_stream(lanes, 0, n)
    t32 = torch.empty(n, dtype=torch.float32, device="cuda")
    V.VmtGenerator(42, V.VmtConfig(8)).fill_f32(t32)
    ref32 = (u >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -24)
    assert np.array_equal(host(t32).view(np.uint32), ref32.view(np.uint32))
    del t32, ref32
    t64 = torch.empty(n, dtype=torch.float64, device="cuda")
    V.VmtGenerator(42, V.VmtConfig(8)).fill_f64(t64)
    ref64 = u.astype(np.float64) * 2.0 ** -32
    assert np.array_equal(host(t64).view(np.uint64), ref64.view(np.uint64))


def test_config3_full_size_every_generator(golden, gnpz):
    """c3 as BASELINE.json states it: 1024 generators (seeds 1..1024), L=16,
    default (full-period) de-phasing, 2^20 words each, generator-major, in one
    batch call. Every generator's XOR fold, first 4 and last words equal the C
    oracle's (tests/golden/c3_full.npz, make_golden.py c3_full), hence the
    full 2^30-word checksum too."""
    n, ngen = 1 << 20, 1024
    ref = gnpz("c3_full.npz")
    out = dev_u32(n * ngen)
    V.batch_fill_u32(out, 1, ngen, 16, n)
    v = host(out).reshape(ngen, n)
    folds = np.bitwise_xor.reduce(v, axis=1)
    assert np.array_equal(folds, ref["folds"])
    assert np.array_equal(v[:, :4], ref["heads"]) and np.array_equal(v[:, -1], ref["lasts"])
    assert int(np.bitwise_xor.reduce(folds)) == golden["c3_full"]["xor"]


@pytest.mark.parametrize("seed", [1, 512, 1024])
def test_config3_sampled_generators_vs_oracle(oracle, full_polys, seed):
    """Sampled c3 generators at q=19933, all 2^20 words against the C oracle:
    from the 1024-generator batch (tensor-core de-phasing) and from a single
    generator (polynomial de-phasing)."""
    n, ngen = 1 << 20, 1024
    ref = oracle_window(oracle, seed, 16, full_polys["q19933"], 0, n)
    out = dev_u32(n * ngen)
    V.batch_fill_u32(out, 1, ngen, 16, n)
    assert np.array_equal(host(out[(seed - 1) * n:seed * n]), ref), seed
    del out
    w = dev_u32(n)
    V.VmtGenerator(seed, V.VmtConfig(16)).fill_u32(w)
    assert np.array_equal(host(w), ref), seed


@pytest.mark.parametrize("L", [8, 16, 32])
def test_float_fills_ragged_and_misaligned(oracle, L):
    """Float32 / float64 fills of ragged lengths into views at odd element
    offsets: consecutive fills start at odd stream positions and write to
    destinations that are not 8- / 16-byte aligned, so both the vector
    (float2 / double2) and the scalar store paths run; every value must equal
    the conversion rule applied to the oracle's stream."""
    q = 16
    sizes = [1001, 2048, 333, 70000 + 3, 1]
    total = sum(sizes)
    lanes = oracle.dephased_states(7, L, oracle.x_pow2_mod(q))
    u = oracle.vmt_stream(lanes, 0, total)
    ref32 = (u >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -24)
    ref64 = (u.astype(np.float64) + 0.5) * 2.0 ** -32
    for kind, ref in (("f32", ref32), ("f64", ref64)):
        g = V.VmtEngine(L, 7, q)
        dt = torch.float32 if kind == "f32" else torch.float64
        buf = torch.empty(total + 2 * len(sizes) + 1, dtype=dt, device="cuda")
        pos, off, views = 0, 1, []
        for k, sz in enumerate(sizes):
            v = buf[off:off + sz]
            if kind == "f32":
                g.fill_f32(v)
            else:
                g.fill_f64(v, rule=V.VMT_F64_REAL3)
            views.append((v, pos, sz))
            pos += sz
            off += sz + (k % 2)  # alternate parity of the next destination
        for v, p0, sz in views:
            assert np.array_equal(host(v), ref[p0:p0 + sz]), (kind, p0, sz)
