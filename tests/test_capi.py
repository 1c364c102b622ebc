"""CPU-side checks of the product boundary: the C-ABI library loads and
exports every symbol include/vmt19937_b200.h declares, the host jump-polynomial
math agrees with the oracle and the golden fixtures, argument validation maps
to the reference's exception classes, and generation refuses to run without a
GPU (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def header_symbols():
    with open(os.path.join(ROOT, "include", "vmt19937_b200.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)  # drop comments
    return sorted(set(re.findall(r"^[A-Za-z_][\w \*]*?\b(vmt_[a-z0-9_]+)\s*\(", text, flags=re.M)))


def test_library_exports_every_header_symbol():
    import paper_2309_16682_b200._capi as capi
    lib = ctypes.CDLL(capi.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(capi.EXPORTS) == syms


def test_library_is_sm100a():
    import subprocess
    import paper_2309_16682_b200._capi as capi
    out = subprocess.run(["cuobjdump", "--list-elf", capi.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_library_links_no_cuda_math_library():
    """Every kernel on the path is ours: the library needs no cuBLAS/cuBLASLt
    (or any other CUDA library; the runtime is linked statically)."""
    import subprocess
    import paper_2309_16682_b200._capi as capi
    out = subprocess.run(["readelf", "-d", capi.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("readelf unavailable")
    needed = [ln.split("[")[1].rstrip("]") for ln in out.stdout.splitlines() if "(NEEDED)" in ln]
    assert needed, out.stdout
    for lib in needed:
        assert not any(x in lib for x in ("cublas", "cudnn", "cufft", "curand", "cusparse", "libcudart")), needed


def test_full_period_exponents():
    import paper_2309_16682_b200 as V
    # jump.cpp:13-15, test_jump.cpp:32-38 (+ L=32)
    assert [V.JumpSpec.full_period_exponent(L) for L in (1, 2, 4, 8, 16, 32)] == [
        19937, 19936, 19935, 19934, 19933, 19932]
    assert V.JumpSpec.full_period_split(16).is_full_period_split()
    assert not V.JumpSpec(10, 16).is_full_period_split()
    with pytest.raises(V.InvalidArgument):
        V.JumpSpec(5, 3).validate()
    assert V.VmtConfig(16).jump_exponent == 19933


def test_charpoly_matches_golden(gnpz):
    import paper_2309_16682_b200 as V
    assert np.array_equal(V.charpoly(), gnpz("charpoly.npy"))


@pytest.mark.parametrize("q", [0, 1, 6, 16, 31, 64, 1000, 4096])
def test_jump_poly_pow2_matches_oracle(oracle, q):
    import paper_2309_16682_b200 as V
    assert np.array_equal(V.jump_poly_pow2(q), oracle.x_pow2_mod(q))


def test_full_period_polys_match_golden(full_polys):
    import paper_2309_16682_b200 as V
    for q in range(19932, 19937):
        assert np.array_equal(V.jump_poly_pow2(q), full_polys[f"q{q}"]), q
    x = np.zeros(312, np.uint64)
    x[0] = 2
    assert np.array_equal(V.jump_poly_pow2(19937), x)  # period
    assert np.array_equal(V.jump_poly_pow2(19937 + 5), V.jump_poly_pow2(5))


@pytest.mark.parametrize("d", [0, 1, 2, 623, 624, 9984, 2**32 + 7, 12345678901234567, 2**64 - 1])
def test_jump_poly_matches_oracle(oracle, d):
    import paper_2309_16682_b200 as V
    assert np.array_equal(V.jump_poly(d), oracle.x_pow_mod(d))


def test_jump_poly_128bit_composes(oracle):
    import paper_2309_16682_b200 as V
    a = V.jump_poly(2**64)  # x^(2^64) = (x^(2^32))^(2^32)
    assert np.array_equal(a, V.jump_poly_pow2(64))
    b = V.jump_poly(2**70 + 5)
    assert np.array_equal(b, oracle.mulmod(V.jump_poly_pow2(70), oracle.x_pow_mod(5)))


def test_invalid_lanes_is_invalid_argument():
    import paper_2309_16682_b200 as V
    for L in (0, 3, 5, 64):
        with pytest.raises(V.InvalidArgument):
            V.VmtGenerator(1, V.VmtConfig(L))


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2309_16682_b200 as V
    with pytest.raises(V.VmtError) as e:
        V.VmtGenerator(5489, V.VmtConfig(16))
    assert e.value.code == -4
    with pytest.raises(V.VmtError):
        V.batch_fill_u32(np.empty(16, np.uint32), 1, 1, 16, 16)
    with pytest.raises(V.VmtError):
        V.jump_states(np.zeros((1, 624), np.uint32), [5])


def test_argument_errors_without_gpu():
    """The C ABI validates arguments before touching the device: the
    reference's std::invalid_argument cases come back as VMT_EINVAL."""
    import ctypes
    import paper_2309_16682_b200 as V
    from paper_2309_16682_b200 import _capi
    lib = _capi.lib
    h = ctypes.c_void_p()
    assert lib.vmt_batch_create(1, 4, 3, 0, 0, ctypes.byref(h)) == _capi.VMT_EINVAL      # lanes
    assert lib.vmt_batch_create(1, 0, 4, 0, 0, ctypes.byref(h)) == _capi.VMT_EINVAL      # ngen
    devs = (ctypes.c_int * 1)(0)
    assert lib.vmt_multi_gpu_fill(1, 4, 0, 10, 1, devs, None, 7, None) == _capi.VMT_EINVAL  # mode
    assert lib.vmt_multi_gpu_fill(1, 4, 0, 10, 1, devs, None, 0, None) == _capi.VMT_EINVAL  # no dsts
    assert lib.vmt_multi_gpu_fill(1, 4, 0, 10, 0, devs, None, 1, None) == _capi.VMT_EINVAL  # ngpus
    out = ctypes.c_double()
    assert lib.vmt_store_bandwidth(0, 1 << 20, 5, 1, ctypes.byref(out)) == _capi.VMT_EINVAL
    assert lib.vmt_create_from_matrix(1, 8, None, 3, 0, ctypes.byref(h)) == _capi.VMT_EINVAL
    assert lib.vmt_vec_mat_mul(None, 1, None, None, 0, None) == _capi.VMT_EINVAL
    assert lib.vmt_jump_states_matrix(None, 1, None, None, 0, None) == _capi.VMT_EINVAL
    assert lib.vmt_create(1, 3, 0, 0, ctypes.byref(h)) == _capi.VMT_EINVAL
    u = ctypes.c_uint64()
    assert lib.vmt_set_prefetch(None, _capi.VMT_PREFETCH_TENSOR) == _capi.VMT_EINVAL
    assert lib.vmt_prefetch_stats(None, ctypes.byref(u), ctypes.byref(u)) == _capi.VMT_EINVAL
    with pytest.raises(V.InvalidArgument):
        V.write_jump_matrix_file("/tmp/never.vmtj", np.zeros(5, np.uint64), 1)
    assert b"invalid" in lib.vmt_status_string(_capi.VMT_EINVAL)


@pytest.mark.parametrize("fill,dt", [("fill_u32", "uint32"), ("fill_f32", "float32"), ("fill_f64", "float64")])
def test_fill_rejects_n_beyond_buffer(fill, dt):
    """Every fill checks n against the destination's size before calling the
    C ABI (which cannot see the buffer's extent)."""
    import numpy as np
    import paper_2309_16682_b200 as V
    g = V.VmtGenerator.__new__(V.VmtGenerator)  # no device needed: the check comes first
    g._h = None
    with pytest.raises(V.InvalidArgument):
        getattr(g, fill)(np.empty(8, dt), n=9)


def test_dist_collective_device_defaults():
    import torch
    from paper_2309_16682_b200 import dist as D
    assert D.collective_device() == torch.device("cpu")  # no process group: CPU
    assert D.collective_device("cuda:3") == torch.device("cuda", 3)
