"""The .vmtj jump-matrix file format (jump_file.hpp:12-22, jump_file.cpp):
the library's host reader/writer against the reference's own reader/writer
(oracle/_ref) and the golden SHA-256 of the reference's files. Host code only,
no GPU (the matrices themselves come from the reference here)."""
import hashlib
import os
import struct

import numpy as np
import pytest

import paper_2309_16682_b200 as V
from paper_2309_16682_b200 import _capi

REF_SO = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "libvmtref.so")


@pytest.fixture(scope="module")
def ref():
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built")
    from oracle import RefLib
    return RefLib()


@pytest.fixture(scope="module")
def ref_file_q2(ref, tmp_path_factory):
    path = str(tmp_path_factory.mktemp("vmtj") / "F_2p2.vmtj")
    ref.write_pow2_matrix_file(2, path)
    return path


def file_sha(path):
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def test_reference_file_matches_golden(ref_file_q2, golden):
    assert file_sha(ref_file_q2) == golden["vmtj"]["2"]["sha256"]


def test_read_reference_file_and_rewrite_identical(ref_file_q2, ref, tmp_path):
    rows, e = V.read_jump_matrix_file(ref_file_q2)
    assert e == 2 and rows.shape == (19937, 312)
    ref_rows, ref_e = ref.read_jump_matrix_file(ref_file_q2)
    assert ref_e == 2 and np.array_equal(rows, ref_rows)
    out = str(tmp_path / V.jump_matrix_file_name(2))
    V.write_jump_matrix_file(out, rows, 2)
    assert file_sha(out) == file_sha(ref_file_q2)
    assert not os.path.exists(out + ".tmp")
    # the reference reads the library's file back
    back, be = ref.read_jump_matrix_file(out)
    assert be == 2 and np.array_equal(back, rows)
    # header-only validation
    assert V.read_jump_matrix_file(out, rows=False) == (None, 2)


def _write(path, magic=b"VMTJ", version=1, dim=19937, exponent=3, reserved=0, payload=None, pad_bit=False):
    words = (dim + 63) // 64
    if payload is None:
        payload = np.zeros(dim * words, np.uint64)
        if pad_bit and dim % 64:
            payload[words - 1] = np.uint64(1) << np.uint64(63)
    with open(path, "wb") as f:
        f.write(magic + struct.pack("<IIII", version, dim, exponent, reserved))
        f.write(np.asarray(payload, np.uint64).tobytes())


@pytest.mark.parametrize("case,kw", [
    ("magic", dict(magic=b"VMTX")),
    ("version", dict(version=2)),
    ("reserved", dict(reserved=7)),
    ("zero_dim", dict(dim=0)),
    ("padding", dict(pad_bit=True)),
])
def test_format_errors_match_reference(tmp_path, ref, case, kw):
    path = str(tmp_path / f"{case}.vmtj")
    _write(path, **kw)
    with pytest.raises(V.VmtError) as ei:
        V.read_jump_matrix_file(path)
    assert ei.value.code == _capi.VMT_EIO
    with pytest.raises(RuntimeError, match="rc=-3"):  # std::runtime_error
        ref.read_jump_matrix_file(path)


def test_truncated_and_missing(tmp_path, ref):
    path = str(tmp_path / "short.vmtj")
    _write(path, payload=np.zeros(19937 * 312 - 1, np.uint64))
    for p in (path, str(tmp_path / "absent.vmtj")):
        with pytest.raises(V.VmtError) as ei:
            V.read_jump_matrix_file(p)
        assert ei.value.code == _capi.VMT_EIO
        with pytest.raises(RuntimeError, match="rc=-3"):
            ref.read_jump_matrix_file(p)


def test_other_dimension_is_invalid_argument(tmp_path, ref):
    """A well-formed 64-dimensional file loads in the reference (F2Matrix is
    any size) but cannot drive a 19937-bit jump: std::invalid_argument, as
    vec_mat_mul's dimension check (f2_matrix.cpp:120-121)."""
    path = str(tmp_path / "small.vmtj")
    _write(path, dim=64)
    rows, e = ref.read_jump_matrix_file(path)
    assert rows.shape == (64, 1) and e == 3
    with pytest.raises(V.InvalidArgument):
        V.read_jump_matrix_file(path)
    with pytest.raises(V.InvalidArgument):
        V.VmtGenerator(5489, V.VmtConfig(4), jump_matrix_file=path)


def test_write_rejects_wrong_size(tmp_path):
    with pytest.raises(V.InvalidArgument):
        V.write_jump_matrix_file(str(tmp_path / "x.vmtj"), np.zeros(10, np.uint64), 1)
