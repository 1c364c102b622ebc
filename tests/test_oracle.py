"""Pins the C oracle (oracle/vmt_oracle.c) against the reference's own KATs
(proj/tests/test_mt19937.cpp, test_jump.cpp, test_engine.cpp) and against the
golden vectors produced by the unmodified reference library
(tests/golden/make_golden.py). CPU only."""
import hashlib

import numpy as np
import pytest

from conftest import dephase_poly


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# --- test_mt19937.cpp KATs ------------------------------------------------

def test_temper_and_mul_a_kats(oracle):
    # test_mt19937.cpp:48-58
    assert oracle.temper(0x00000000) == 0x00000000
    assert oracle.temper(0x00000001) == 0x00400091
    assert oracle.temper(0xFFFFFFFF) == 0x6FE01BF8
    assert oracle.mul_a(0) == 0
    assert oracle.mul_a(1) == 0x9908B0DF
    assert oracle.mul_a(3) == 0x9908B0DE


def test_mul_a_companion_matrix(oracle):
    # test_mt19937.cpp:60-76
    rows = [0x9908B0DF] + [1 << (i - 1) for i in range(1, 32)]
    for u in oracle.mt64(7, 1000):
        u = int(u) & 0xFFFFFFFF
        prod = 0
        for i in range(32):
            if (u >> i) & 1:
                prod ^= rows[i]
        assert oracle.mul_a(u) == prod


def test_seeding_and_first_outputs(oracle, golden):
    w = oracle.seed_words(5489)
    assert w[0] == 5489 and w[1] == 1301868182 == golden["seed5489_word1"]
    assert list(oracle.mt_stream(5489, 3)) == [3499211612, 581869302, 3890346734] == golden["seed5489_first3"]
    assert np.any(oracle.seed_words(0)[1:] != 0)


def test_scalar_10k_matches_reference(oracle, golden):
    for seed, g in golden["scalar10k"].items():
        v = oracle.mt_stream(int(seed), 10000)
        assert sha(v) == g["sha"] and int(v[-1]) == g["last"]


def test_scalar_skip_consistency(oracle):
    full = oracle.mt_stream(42, 5000)
    for skip in (0, 1, 623, 624, 625, 1248, 3001):
        assert np.array_equal(oracle.mt_stream(42, 100, skip=skip), full[skip:skip + 100])


def test_std_mt19937_64_seed7(oracle, gnpz):
    # the tests' RNG idiom (test_mt19937.cpp:67); distances of config 5
    assert np.array_equal(oracle.mt64(7, 8), gnpz("c5_ref.npz")["dists"])


# --- matrix jump (f2_matrix.cpp / jump.cpp) ---------------------------------

def test_transition_matrix_step_equals_reference(oracle, gnpz):
    F = oracle.transition_matrix()
    s = oracle.seed_words(5489)
    assert np.array_equal(oracle.jump_state_matrix(s, F), gnpz("ref_jumps.npz")["q0"])


def test_matrix_square_equals_two_steps(oracle):
    F = oracle.transition_matrix()
    F2 = oracle.mat_mul(F, F)
    s = oracle.seed_words(777)
    once = oracle.jump_state_matrix(oracle.jump_state_matrix(s, F), F)
    assert np.array_equal(oracle.jump_state_matrix(s, F2), once)


# --- polynomial jump (G3) pinned to the reference matrix jump ---------------

def test_charpoly(oracle, gnpz):
    P = oracle.charpoly()
    assert np.array_equal(P, gnpz("charpoly.npy"))
    assert int(P[0]) & 1 == 1  # x does not divide P
    # P annihilates every word sequence: sum_j p_j x_{n+j} == 0
    x = oracle.mt_stream(0, 0)
    s = oracle.seed_words(2024)
    seq = np.empty(19937 + 624 + 64, np.uint32)
    seq[:624] = s
    ua = np.uint32(0x80000000)
    la = np.uint32(0x7FFFFFFF)
    for n in range(seq.size - 624):
        u = (seq[n] & ua) | (seq[n + 1] & la)
        seq[n + 624] = seq[n + 397] ^ (u >> np.uint32(1)) ^ (np.uint32(0x9908B0DF) if u & 1 else np.uint32(0))
    bits = np.unpackbits(P.view(np.uint8), bitorder="little")[:19938].astype(bool)
    idx = np.nonzero(bits)[0]
    for n in (1, 7, 50):
        acc = np.bitwise_xor.reduce(seq[n + idx])
        assert acc == 0


@pytest.mark.parametrize("q", [0, 4, 8, 10, 11, 16])
def test_poly_jump_equals_reference_matrix_jump(oracle, gnpz, q):
    s = oracle.seed_words(5489)
    assert np.array_equal(oracle.poly_jump(s, oracle.x_pow2_mod(q)), gnpz("ref_jumps.npz")[f"q{q}"])


def test_jump_skips_exactly_d_outputs(oracle):
    # test_jump.cpp:53-64, at non-power-of-two distances too
    s = oracle.seed_words(5489)
    ref = oracle.mt_stream(5489, 1000, skip=0)
    for d in (1, 5, 624, 1000, 123457):
        j = oracle.poly_jump(s, oracle.x_pow_mod(d))
        assert np.array_equal(oracle.mt_stream_from_words(j, 500), oracle.mt_stream(5489, 500, skip=d))
    assert ref.size == 1000


def test_full_period_polys_and_period_identity(oracle, full_polys):
    # x^(2^19937) == x mod P (period 2^19937 - 1) and sqrt chain consistency
    x = np.zeros(312, np.uint64)
    x[0] = 2
    q36 = full_polys["q19936"]
    out = np.empty(312, np.uint64)
    oracle.lib.or_poly_sqrmod(q36, oracle.charpoly(), out)
    assert np.array_equal(out, x)
    for q in range(19932, 19936):
        oracle.lib.or_poly_sqrmod(full_polys[f"q{q}"], oracle.charpoly(), out)
        assert np.array_equal(out, full_polys[f"q{q + 1}"])


@pytest.mark.parametrize("L", [8, 16, 32])
def test_full_period_lanes_wrap_to_one_step(oracle, full_polys, L):
    # L jumps of 2^q with L*2^q = 2^19937 == one step (SURVEY.md 8c pin 2)
    q = 19937 - (L.bit_length() - 1)
    s = oracle.seed_words(5489)
    v = s.copy()
    for _ in range(L):
        v = oracle.poly_jump(v, full_polys[f"q{q}"])
    one = oracle.poly_jump(s, oracle.x_pow_mod(1))
    assert np.array_equal(v, one)
    assert np.array_equal(oracle.mt_stream_from_words(v, 100), oracle.mt_stream(5489, 100, skip=1))


# --- VMT engine streams (engine.hpp) ----------------------------------------

def test_engine_streams_match_reference(oracle, golden, gnpz):
    streams = gnpz("engine_streams.npz")
    polys = {}
    for e in golden["engine"]:
        L, q, seed = e["lanes"], e["q"], e["seed"]
        if q not in polys:
            polys[q] = oracle.x_pow2_mod(q)
        lanes = oracle.dephased_states(seed, L, polys[q])
        v = oracle.vmt_stream(lanes, 0, e["count"])
        assert sha(v) == e["sha"], (L, q, seed)
        assert np.array_equal(v[:4096], streams[f"L{L}_q{q}_s{seed}"])


def test_appendix_a_checksums(oracle, golden):
    for row in golden["appendixA"]:
        L, seed, q, n = row["lanes"], row["seed"], row["q"], row["count"]
        lanes = oracle.dephased_states(seed, L, oracle.x_pow2_mod(q)) if L > 1 else oracle.seed_words(seed)[None]
        assert oracle.vmt_checksum(lanes, 0, n) == row["xor"], row
        assert list(oracle.vmt_stream(lanes, 0, 4)) == row["first4"]
        assert int(oracle.vmt_stream(lanes, n - 1, 1)[0]) == row["last"]


def test_interleave_identity(oracle):
    # output[i*M + t] == scalar[t*2^q + i] (test_engine.cpp:37-49)
    for L, q in ((2, 6), (4, 8), (8, 6), (16, 8), (32, 6)):
        w = 1 << q
        scalar = oracle.mt_stream(5489, w * L)
        v = oracle.vmt_stream(oracle.dephased_states(5489, L, oracle.x_pow2_mod(q)), 0, w * L)
        assert np.array_equal(v.reshape(w, L).T.reshape(-1), scalar)


def test_lane_independence_after_three_blocks(oracle, gnpz):
    # test_engine.cpp:137-158
    lanes = oracle.dephased_states(31337, 4, oracle.x_pow2_mod(10))
    s = np.empty(624 * 4, np.uint32)
    oracle.lib.or_vmt_interleave = oracle.lib.or_vmt_interleave
    il = lanes.T.reshape(-1).copy()
    for _ in range(3):
        oracle.lib.or_vmt_regenerate(il, 4)
    assert np.array_equal(il, gnpz("engine_state_L4_q10_s31337_b3.npy"))
    assert s.size == 2496


def test_dephased_L32_matches_reference(oracle, gnpz):
    ref = gnpz("ref_jumps.npz")["dephased_L32_q16_s5489"]
    assert np.array_equal(oracle.dephased_states(5489, 32, oracle.x_pow2_mod(16)), ref)


def test_config4_windows_q16(oracle, golden):
    """The window helper the full-period GPU tests use (conftest.oracle_window)
    reproduces the reference's own windows (rung composition through
    jump_state, make_golden.py) at q=16."""
    from conftest import oracle_window
    lanes = oracle.dephased_states(5489, 32, oracle.x_pow2_mod(16))
    for w in golden["c4_windows_q16"]:
        v = oracle_window(oracle, 5489, 32, None, w["start_word"], w["count"], dephased=lanes)
        assert sha(v) == w["sha"] and list(v[:8]) == w["head"]


def test_oracle_window_unaligned_start(oracle):
    """oracle_window at a start inside a block equals the plain stream."""
    from conftest import oracle_window
    poly = oracle.x_pow2_mod(8)
    full = oracle.vmt_stream(oracle.dephased_states(7, 16, poly), 0, 5 * 624 * 16 + 3000)
    for start in (1, 624 * 16 - 1, 3 * 624 * 16 + 17):
        assert np.array_equal(oracle_window(oracle, 7, 16, poly, start, 3000), full[start:start + 3000])


def test_c3_full_fixture_consistent(golden, gnpz):
    ref = gnpz("c3_full.npz")
    assert ref["folds"].shape == (1024,) and ref["heads"].shape == (1024, 4)
    assert int(np.bitwise_xor.reduce(ref["folds"])) == golden["c3_full"]["xor"]



def test_c3_first_outputs_are_scalar_first_outputs(oracle, gnpz):
    """Output[0] of every c3 generator is its seed's first scalar MT output
    (independent of the de-phasing)."""
    heads = gnpz("c3_full.npz")["heads"]
    for s in range(1, 1025):
        assert int(heads[s - 1, 0]) == int(oracle.mt_stream(s, 1)[0]), s


def test_config5_jumps_match_reference(oracle, gnpz):
    c5 = gnpz("c5_ref.npz")
    for i, d in enumerate(c5["dists"]):
        s = oracle.seed_words(i + 1)
        j = oracle.poly_jump(s, oracle.x_pow_mod(int(d)))
        assert np.array_equal(oracle.mt_stream_from_words(j, 624), c5[f"s{i + 1}"])


def test_bench_checksums_mode_invariant(oracle, golden):
    by = {}
    for r in golden["bench_checksums"]:
        by.setdefault(r["lanes"], set()).add(r["xor"])
    for L, xs in by.items():
        assert len(xs) == 1  # identical across single / block16 / state (test_cli.cpp:105-118)
        lanes = oracle.dephased_states(5489, L, oracle.x_pow2_mod(6)) if L > 1 else oracle.seed_words(5489)[None]
        assert oracle.vmt_checksum(lanes, 0, 1000000) == next(iter(xs))
