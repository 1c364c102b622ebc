"""GPU parity of the fused statistics consumer (north_star "optional fused
consumer (checksum or histogram)"): one-bit and byte-value
counts taken inside the generation kernel (nothing stored) against the
reference's stream, and monobit / chi2_bytes reports against the reference's
stats.cpp on the same streams."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2309_16682_b200 as V  # noqa: E402

POP8 = np.array([bin(i).count("1") for i in range(256)], np.uint64)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")


def np_counts(words):
    bins = np.bincount(np.asarray(words, np.uint32).view(np.uint8), minlength=256).astype(np.uint64)
    return int((bins * POP8).sum()), bins


def test_counts_and_reports_match_reference(golden):
    for c in golden["stats"]["reports"]:
        g = V.VmtGenerator(c["seed"], V.VmtConfig(c["lanes"], jump_exponent=c["q"]))
        ones, bins = g.stat_counts(c["count"])
        assert ones == c["ones"], c
        assert [int(b) for b in bins] == c["bins"], c
        for fn, name in ((V.monobit, "monobit"), (V.chi2_bytes, "chi2_bytes")):
            r = fn(V.VmtGenerator(c["seed"], V.VmtConfig(c["lanes"], jump_exponent=c["q"])), c["count"])
            ref = c[name]
            assert r.name == name and r.samples == c["count"]
            assert r.statistic == ref["statistic"], (name, c["lanes"], r.statistic, ref["statistic"])
            assert r.p_value == ref["p_value"], (name, c["lanes"])
            assert r.pass_ == ref["pass"], (name, c["lanes"])


def test_counts_continue_the_stream(oracle):
    """Counting consumes words like a fill: mixed with next_u32 / fills and at
    ragged positions the counted words are exactly the next n of the stream."""
    L, q = 16, 12
    lanes = oracle.dephased_states(9, L, oracle.x_pow2_mod(q))
    total = 3 * 624 * L + 777
    ref = oracle.vmt_stream(lanes, 0, total + 200000)
    g = V.VmtEngine(L, 9, q)
    pos = 0
    for _ in range(5):
        assert g.next_u32() == ref[pos]
        pos += 1
    for n in (13, 624 * L - 1, 2 * 624 * L + 5, 100003):
        ones, bins = g.stat_counts(n)
        eo, eb = np_counts(ref[pos:pos + n])
        assert ones == eo and np.array_equal(bins, eb), n
        pos += n
    out = np.empty(50, np.uint32)
    g.fill_u32(out)
    assert np.array_equal(out, ref[pos:pos + 50])


def test_undersized_samples_rejected():
    g = V.VmtEngine(4, 1, 8)
    with pytest.raises(V.InvalidArgument):
        V.monobit(g, 999999)
    with pytest.raises(V.InvalidArgument):
        V.chi2_bytes(g, 3199)


@pytest.mark.parametrize("L", [8, 32])
def test_large_counts_vs_stored_stream(L):
    """At 2^30 words: the fused counts equal a torch bincount of the same words
    stored by fill_u32 (size-independent check of the histogram path)."""
    n = 1 << 30
    g = V.VmtGenerator(5489, V.VmtConfig(L))
    ones, bins = g.stat_counts(n)
    h = V.VmtGenerator(5489, V.VmtConfig(L))
    buf = torch.empty(n, dtype=torch.uint32, device="cuda")
    h.fill_u32(buf)
    tb = torch.bincount(buf.view(torch.uint8), minlength=256).cpu().numpy().astype(np.uint64)
    del buf
    assert np.array_equal(bins, tb)
    assert ones == int((tb * POP8).sum())
    assert int(bins.sum()) == 4 * n


def test_lane_cross_correlation_matches_reference(golden):
    """Floating point: the reference's own build mixes vectorised and fused
    sums, so parity is within 1e-12 relative (statistic and p-value)."""
    for c in golden["stats"]["lane_corr"]:
        g = V.VmtGenerator(c["seed"], V.VmtConfig(c["lanes"], jump_exponent=c["q"]))
        r = V.lane_cross_correlation(g, c["count"])
        assert r.name == "lane_cross_correlation" and r.samples == c["count"]
        assert r.statistic == pytest.approx(c["statistic"], rel=1e-12), c
        assert r.p_value == pytest.approx(c["p_value"], rel=1e-9), c
        assert r.pass_ == c["pass"]
    with pytest.raises(V.InvalidArgument):
        V.lane_cross_correlation(V.VmtGenerator(1, V.VmtConfig(1)), 1000)


@pytest.mark.parametrize("L", [8, 16, 32])
def test_counts_long_chunks_match_stored_words(L):
    """Long chunks (max_chunks=8 at 2^28 words: 6721 / 3360 / 1680 blocks per
    chunk for L = 8 / 16 / 32, far past any 16-bit count): the fused counts
    equal a byte histogram of the same stored words (torch.bincount on the
    GPU), and the one-bit count their popcount."""
    n = 1 << 28
    a = V.VmtGenerator(77, V.VmtConfig(L))
    a.set_tuning(max_chunks=8)
    ones, bins = a.stat_counts(n)
    b = V.VmtGenerator(77, V.VmtConfig(L))
    out = torch.empty(n, dtype=torch.uint32, device="cuda")
    b.fill_u32(out)
    ref = torch.bincount(out.view(torch.uint8).to(torch.int64), minlength=256).cpu().numpy().astype(np.uint64)
    assert np.array_equal(np.asarray(bins, np.uint64), ref)
    assert ones == int((ref * POP8).sum())
    assert int(ref.sum()) == 4 * n
