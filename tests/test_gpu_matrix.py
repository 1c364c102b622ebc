"""GPU parity of the GF(2) jump-matrix path: jump
matrices computed on the GPU against the reference's .vmtj bytes (golden
SHA-256 from its squaring ladder), vec_mat_mul against numpy, matrix
de-phasing against the reference's make_dephased_states, and full-period
matrix properties where the reference cannot compute the matrix (~50 h)."""
import hashlib
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2309_16682_b200 as V  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")


def file_sha(path):
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def np_vec_mat(vecs, rows):
    """vec_mat_mul restated in numpy: XOR of the rows at the set bits."""
    out = np.zeros_like(vecs)
    for s, v in enumerate(vecs):
        bits = np.unpackbits(v.view(np.uint8), bitorder="little")[:19937].astype(bool)
        if bits.any():
            out[s] = np.bitwise_xor.reduce(rows[bits], axis=0)
    return out


def words_to_eff(w):
    """state_to_effective (mt19937.cpp:57-101) in numpy."""
    w = np.asarray(w, np.uint32)
    nxt = np.concatenate([w[1:], np.zeros(1, np.uint32)])
    e32 = (w >> np.uint32(31)) | (nxt << np.uint32(1))
    return e32.view(np.uint64)


@pytest.mark.parametrize("q", [0, 1, 2, 5, 10, 16, 20, 24])
def test_pow2_matrix_file_bytes_match_reference(golden, tmp_path, q):
    """compute_jump_matrix (jump_file.cpp:171-209): the file the GPU writes for
    F^(2^q) is byte-identical to the reference's mat_pow2 ladder output."""
    path = str(tmp_path / V.jump_matrix_file_name(q))
    V.compute_jump_matrix(q, path)
    g = golden["vmtj"][str(q)]
    if file_sha(path) != g["sha256"]:
        rows, e = V.read_jump_matrix_file(path)
        assert e == q
        assert [int(v) for v in rows[0, :4]] == g["row0"], "row 0"
        assert [int(v) for v in rows[-1, -4:]] == g["row19936"], "row 19936"
        assert int(np.bitwise_xor.reduce(rows, axis=None)) == g["row_xor_fold"], "row fold"
        pytest.fail("file bytes differ")
    assert os.path.getsize(path) == g["size"]


def test_device_matrix_equals_host_matrix():
    rows_h = V.jump_matrix_pow2(10)
    rows_d = torch.empty((19937, 312), dtype=torch.uint64, device="cuda")
    V.jump_matrix_pow2(10, out=rows_d)
    torch.cuda.synchronize()
    assert np.array_equal(rows_d.cpu().numpy(), rows_h)
    # F^1 is the transition matrix, F^(2^1) = F^2
    assert np.array_equal(V.jump_matrix(1), V.jump_matrix_pow2(0))
    assert np.array_equal(V.jump_matrix(2), V.jump_matrix_pow2(1))


def test_vec_mat_mul_batched_vs_numpy():
    rows = V.jump_matrix(123456789)
    rng = np.random.default_rng(5)
    vecs = rng.integers(0, 2**63, size=(9, 312), dtype=np.uint64)  # 9: not a multiple of the CTA batch
    vecs[:, -1] &= np.uint64((1 << 33) - 1)
    vecs[3] = 0
    got = V.vec_mat_mul(vecs, rows)
    assert np.array_equal(got, np_vec_mat(vecs, rows))


def test_jump_state_matrix_matches_reference(gnpz):
    """jump_state(seed 5489, F^(2^q)) (jump.cpp:27-33) for the reference's rungs."""
    jumps = gnpz("ref_jumps.npz")
    s0 = V.seed_states(np.array([5489], np.uint32))[0]
    for q in (0, 4, 8, 10, 11, 16):
        got = V.jump_state_matrix(s0, V.jump_matrix_pow2(q))[0]
        assert np.array_equal(got, jumps[f"q{q}"]), q


def test_matrix_dephasing_matches_reference(gnpz):
    """make_dephased_states with the GPU-built F^(2^16) (lane t = lane t-1 * B)
    equals the reference's lanes, and the matrix-built generator emits the
    same stream as the polynomial-built one."""
    jumps = gnpz("ref_jumps.npz")
    ref = jumps["dephased_L32_q16_s5489"]  # (32, 624), lane-major
    B = V.jump_matrix_pow2(16)
    g = V.VmtGenerator(5489, V.VmtConfig(32, jump_exponent=16), jump_matrix=B)
    st0 = g.interleaved_state()
    assert np.array_equal(st0.reshape(624, 32).T, ref)
    p = V.VmtEngine(32, 5489, 16)
    a, b = torch.empty(1 << 22, dtype=torch.uint32, device="cuda"), torch.empty(1 << 22, dtype=torch.uint32,
                                                                                 device="cuda")
    g.fill_u32(a)
    p.fill_u32(b)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    # the device-resident matrix works the same
    Bd = torch.from_numpy(B.view(np.int64)).cuda().view(torch.uint64)
    g2 = V.VmtGenerator(5489, V.VmtConfig(32, jump_exponent=16), jump_matrix=Bd)
    assert np.array_equal(g2.interleaved_state(), st0)


def test_create_from_file_adopts_exponent(tmp_path, gnpz):
    path = str(tmp_path / V.jump_matrix_file_name(16))
    V.compute_jump_matrix(16, path)
    g = V.VmtGenerator(1, V.VmtConfig(16), jump_matrix_file=path)
    assert g.jump_exponent() == 16
    ref = gnpz("ref_jumps.npz")["dephased_L16_q16_s1"]
    assert np.array_equal(g.interleaved_state().reshape(624, 16).T, ref)


@pytest.mark.parametrize("L", [16, 32])
def test_full_period_matrix_properties(L):
    """B = F^(2^q) at the full-period exponent q = 19937 - log2 L (no reference
    matrix exists: ~50 h of squarings). Pinned by (1) B^L = F^(2^19937) = F
    (the period is 2^19937 - 1) on random effective vectors, (2) the matrix
    de-phasing equals the polynomial de-phasing, and (3) B's rows are the
    effective images of basis states under the polynomial jump."""
    q = 19937 - (L.bit_length() - 1)
    B = V.jump_matrix_pow2(q)
    F = V.jump_matrix_pow2(0)
    rng = np.random.default_rng(L)
    v = rng.integers(0, 2**63, size=(4, 312), dtype=np.uint64)
    v[:, -1] &= np.uint64((1 << 33) - 1)
    w = v
    for _ in range(L):
        w = V.vec_mat_mul(w, B)
    assert np.array_equal(w, V.vec_mat_mul(v, F))
    gm = V.VmtGenerator(5489, V.VmtConfig(L), jump_matrix=B)
    gp = V.VmtGenerator(5489, V.VmtConfig(L))
    assert gm.jump_exponent() == gp.jump_exponent() == q
    assert np.array_equal(gm.interleaved_state(), gp.interleaved_state())
    lane1 = gp.interleaved_state().reshape(624, L).T[1]
    seed = V.seed_states(np.array([5489], np.uint32))[0]
    assert np.array_equal(words_to_eff(lane1), V.vec_mat_mul(words_to_eff(seed)[None], B)[0])
