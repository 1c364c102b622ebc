"""B200-native VMT19937 (arXiv 2309.16682): host-side mirror of the reference
generator interface over the C ABI (include/vmt19937_b200.h).

Reference names are kept (proj/include/vmt19937/engine.hpp, jump.hpp):

* ``JumpSpec``      jump.hpp:13-21 (full_period_exponent: jump.cpp:13-15)
* ``QueryMode``     engine.hpp:15
* ``VmtConfig``     engine.hpp:18-33 (lanes 1..32; 32 lifts engine.hpp:29-32, G1)
* ``VmtGenerator``  engine.hpp:160-207; ``VmtEngine(lanes, seed, q)`` is the
  fixed-lane spelling of engine.hpp:41-68
* ``next_u32 / next_block16 / next_block_state / interleaved_state`` engine.hpp:70-101
* new: ``fill_u32 / fill_f32 / fill_f64 / checksum_xor / skip`` (bulk GPU
  output, any length), ``batch_fill_u32`` (config 3), ``jump_states`` (config 5)

Buffers may be torch tensors (CUDA or CPU) or numpy arrays. Every word is
produced by the sm_100a kernels; there is no CPU generation path.
"""
from __future__ import annotations

import ctypes
import enum
from typing import Optional

import numpy as np

from . import _capi
from ._capi import (VMT_F32_24, VMT_F64_32, VMT_F64_RES53, VMT_F64_REAL3, VMT_FULL_PERIOD,
                    InvalidArgument, LogicError, VmtError, check, lib)

__all__ = [
    "JumpSpec", "QueryMode", "VmtConfig", "VmtGenerator", "VmtEngine", "batch_fill_u32",
    "jump_states", "seed_states", "charpoly", "jump_poly", "jump_poly_pow2", "VmtError",
    "InvalidArgument", "LogicError", "VMT_F32_24", "VMT_F64_32", "VMT_F64_REAL3", "VMT_F64_RES53",
    "KEFFECTIVE_BITS", "KSTATE_LEN", "MATRIX_DIM", "MATRIX_ROW_WORDS", "jump_matrix", "jump_matrix_pow2",
    "write_jump_matrix_file", "read_jump_matrix_file", "compute_jump_matrix", "jump_matrix_file_name",
    "vec_mat_mul", "jump_state_matrix", "StatReport", "monobit", "chi2_bytes", "stat_counts",
    "regularized_gamma_q", "K_SIGNIFICANCE", "lane_cross_correlation", "monobit_from_counts",
    "chi2_bytes_from_counts", "VmtBatch", "multi_gpu_fill", "store_bandwidth", "release_caches",
]

KSTATE_LEN = 624
KEFFECTIVE_BITS = 19937
MATRIX_DIM = 19937
MATRIX_ROW_WORDS = 312
MATRIX_WORDS = MATRIX_DIM * MATRIX_ROW_WORDS


class QueryMode(enum.IntEnum):
    kSingle = 0
    kBlock16 = 1
    kStateBlock = 2


class JumpSpec:
    """Stream splitting: lane t de-phased by t * 2^exponent (jump.hpp:13-21)."""

    def __init__(self, exponent: int, lanes: int):
        self.exponent = exponent
        self.lanes = lanes

    def validate(self) -> None:
        if self.lanes < 1 or (self.lanes & (self.lanes - 1)):
            raise InvalidArgument(_capi.VMT_EINVAL, "lanes must be a power of two")

    @staticmethod
    def full_period_exponent(lanes: int) -> int:
        return int(lib.vmt_full_period_exponent(lanes))

    def is_full_period_split(self) -> bool:
        return self.exponent == self.full_period_exponent(self.lanes)

    @classmethod
    def full_period_split(cls, lanes: int) -> "JumpSpec":
        s = cls(cls.full_period_exponent(lanes), lanes)
        s.validate()
        return s


class VmtConfig:
    """engine.hpp:18-33; jump_exponent defaults to the full-period split."""

    def __init__(self, lanes: int, mode: QueryMode = QueryMode.kSingle, jump_exponent: Optional[int] = None):
        self.lanes = lanes
        self.mode = mode
        self.jump_exponent = JumpSpec.full_period_exponent(lanes) if jump_exponent is None else jump_exponent

    def validate(self) -> None:
        if self.lanes not in (1, 2, 4, 8, 16, 32):
            raise InvalidArgument(_capi.VMT_EINVAL, "lanes must be one of 1, 2, 4, 8, 16, 32")


def _ptr(buf) -> tuple[int, object, int, str]:
    """(address, keepalive, element count, kind) of a torch tensor / numpy array."""
    try:
        import torch  # noqa: F401
        if isinstance(buf, torch.Tensor):
            if not buf.is_contiguous():
                raise InvalidArgument(_capi.VMT_EINVAL, "buffer must be contiguous")
            return buf.data_ptr(), buf, buf.numel(), ("cuda" if buf.is_cuda else "cpu")
    except ImportError:
        pass
    if isinstance(buf, np.ndarray):
        if not buf.flags["C_CONTIGUOUS"]:
            raise InvalidArgument(_capi.VMT_EINVAL, "buffer must be contiguous")
        return buf.ctypes.data, buf, buf.size, "cpu"
    raise InvalidArgument(_capi.VMT_EINVAL, f"unsupported buffer type {type(buf)!r}")


def _stream_for(kind: str, stream) -> Optional[int]:
    if stream is not None:
        return int(stream)
    if kind == "cuda":
        import torch
        s = torch.cuda.current_stream().cuda_stream
        # torch's default stream is the legacy NULL stream; NULL in the C ABI
        # means "the handle's own stream", so name the legacy stream explicitly
        return s if s else CUDA_STREAM_LEGACY
    return None


CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy


def _check_dtype(buf, np_dtype, torch_name: str) -> None:
    dt = getattr(buf, "dtype", None)
    if isinstance(buf, np.ndarray):
        if buf.dtype != np_dtype:
            raise InvalidArgument(_capi.VMT_EINVAL, f"expected {np.dtype(np_dtype)} buffer")
    else:
        if str(dt) != f"torch.{torch_name}":
            raise InvalidArgument(_capi.VMT_EINVAL, f"expected torch.{torch_name} buffer, got {dt}")


class VmtGenerator:
    """Runtime-lane-count VMT19937 generator on one GPU (engine.hpp:160-207)."""

    def __init__(self, seed: int, cfg: Optional[VmtConfig] = None, device: int = 0, *, lane_states=None,
                 jump_matrix=None, jump_matrix_file: Optional[str] = None):
        """``jump_matrix`` (19937 x 312 uint64 rows, host or device) or
        ``jump_matrix_file`` (.vmtj) de-phase with a GF(2) matrix like the
        reference's VmtGenerator(seed, cfg, F2Matrix) (engine.hpp:162-167); the
        file's exponent is adopted. Otherwise the polynomial jump is used."""
        self._h = ctypes.c_void_p()
        if jump_matrix_file is not None:
            cfg = cfg or VmtConfig(1)
            cfg.validate()
            check(lib.vmt_create_from_file(seed & 0xFFFFFFFF, cfg.lanes, str(jump_matrix_file).encode(), device,
                                           ctypes.byref(self._h)))
            self.cfg = VmtConfig(cfg.lanes, cfg.mode, int(lib.vmt_jump_exponent(self._h)))
        elif jump_matrix is not None:
            cfg = cfg or VmtConfig(1)
            cfg.validate()
            addr, keep, n, _ = _ptr(jump_matrix)
            if n != MATRIX_WORDS:
                raise InvalidArgument(_capi.VMT_EINVAL, f"jump matrix must have {MATRIX_WORDS} uint64 words")
            check(lib.vmt_create_from_matrix(seed & 0xFFFFFFFF, cfg.lanes, addr, cfg.jump_exponent, device,
                                             ctypes.byref(self._h)))
            self.cfg = cfg
        elif lane_states is not None:
            arr = np.ascontiguousarray(lane_states, dtype=np.uint32)
            lanes = arr.size // KSTATE_LEN
            check(lib.vmt_create_from_states(arr.ctypes.data, lanes, device, ctypes.byref(self._h)))
            self.cfg = VmtConfig(lanes, QueryMode.kSingle, 0)
        else:
            cfg = cfg or VmtConfig(1)
            cfg.validate()
            self.cfg = cfg
            check(lib.vmt_create(seed & 0xFFFFFFFF, cfg.lanes, cfg.jump_exponent, device, ctypes.byref(self._h)))
        self.device = device

    # -- lifetime -------------------------------------------------------------
    def close(self) -> None:
        if self._h:
            check(lib.vmt_destroy(self._h))
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- reference properties -------------------------------------------------
    @property
    def lanes(self) -> int:
        return int(lib.vmt_lanes(self._h))

    @property
    def state_words(self) -> int:
        return int(lib.vmt_state_words(self._h))

    buffer_words = 16

    def jump_exponent(self) -> int:
        return int(lib.vmt_jump_exponent(self._h))

    @property
    def position(self) -> int:
        return int(lib.vmt_position(self._h))

    # -- reference queries (engine.hpp:70-98) ---------------------------------
    def next_u32(self) -> int:
        v = ctypes.c_uint32()
        check(lib.vmt_next_u32(self._h, ctypes.byref(v)))
        return v.value

    def next_block16(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        out = np.empty(16, np.uint32) if out is None else out
        check(lib.vmt_next_block16(self._h, out.ctypes.data))
        return out

    def next_block_state(self, out=None):
        out = np.empty(self.state_words, np.uint32) if out is None else out
        addr, _, n, _ = _ptr(out)
        if n < self.state_words:
            raise InvalidArgument(_capi.VMT_EINVAL, "buffer smaller than state_words")
        check(lib.vmt_next_block_state(self._h, addr))
        return out

    def interleaved_state(self) -> np.ndarray:
        out = np.empty(self.state_words, np.uint32)
        check(lib.vmt_export_state(self._h, out.ctypes.data))
        return out

    # -- bulk GPU output ------------------------------------------------------
    def fill_u32(self, out, n: Optional[int] = None, stream=None):
        addr, keep, size, kind = _ptr(out)
        _check_dtype(out, np.uint32, "uint32")
        n = size if n is None else n
        if n > size:
            raise InvalidArgument(_capi.VMT_EINVAL, "n exceeds buffer size")
        check(lib.vmt_fill_u32(self._h, addr, n, _stream_for(kind, stream)))
        return out

    def fill_f32(self, out, n: Optional[int] = None, rule: int = VMT_F32_24, stream=None):
        addr, keep, size, kind = _ptr(out)
        _check_dtype(out, np.float32, "float32")
        n = size if n is None else n
        if n > size:
            raise InvalidArgument(_capi.VMT_EINVAL, "n exceeds buffer size")
        check(lib.vmt_fill_f32(self._h, addr, n, rule, _stream_for(kind, stream)))
        return out

    def fill_f64(self, out, n: Optional[int] = None, rule: int = VMT_F64_32, stream=None):
        addr, keep, size, kind = _ptr(out)
        _check_dtype(out, np.float64, "float64")
        n = size if n is None else n
        if n > size:
            raise InvalidArgument(_capi.VMT_EINVAL, "n exceeds buffer size")
        check(lib.vmt_fill_f64(self._h, addr, n, rule, _stream_for(kind, stream)))
        return out

    def checksum_xor(self, n: int, stream=None) -> int:
        v = ctypes.c_uint32()
        check(lib.vmt_checksum_xor(self._h, n, ctypes.byref(v), None if stream is None else int(stream)))
        return v.value

    def synchronize(self) -> None:
        check(lib.vmt_synchronize(self._h))

    def skip(self, d: int) -> None:
        check(lib.vmt_skip(self._h, d))

    def seek(self, pos: int) -> None:
        check(lib.vmt_seek(self._h, pos))

    def set_tuning(self, max_chunks: int = 0, variant: int = 0) -> None:
        check(lib.vmt_set_tuning(self._h, max_chunks, variant))

    def set_prefetch(self, mode: int = _capi.VMT_PREFETCH_TENSOR) -> None:
        """Positioning prefetch of the predicted next fill: 0 off, 1 (or True)
        polynomial jumps on a side stream, 2 the tcgen05 GEMM beside the
        generation kernel (what a new generator starts with)."""
        check(lib.vmt_set_prefetch(self._h, int(mode)))

    def prefetch_stats(self) -> dict:
        t, u = ctypes.c_uint64(), ctypes.c_uint64()
        check(lib.vmt_prefetch_stats(self._h, ctypes.byref(t), ctypes.byref(u)))
        return {"tensor_prefetches": t.value, "used": u.value}

    def set_positioning(self, mode: int = 0) -> None:
        """0 auto (GEMM for repeating fill shapes), 1 polynomial jumps, 2 GEMM."""
        check(lib.vmt_set_positioning(self._h, mode))

    def positioning_stats(self) -> dict:
        g, m = ctypes.c_uint64(), ctypes.c_uint64()
        check(lib.vmt_positioning_stats(self._h, ctypes.byref(g), ctypes.byref(m)))
        return {"gemm_positionings": g.value, "cached_matrices": m.value}

    def set_profiling(self, enable: bool = True) -> None:
        check(lib.vmt_set_profiling(self._h, int(enable)))

    def last_timings(self) -> tuple[float, float]:
        """(jump_ms, gen_ms) of the most recent fill (profiling enabled)."""
        a, b = ctypes.c_float(), ctypes.c_float()
        check(lib.vmt_last_timings(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def stat_counts(self, n: int, stream=None) -> tuple[int, np.ndarray]:
        """Consumes the next n words without storing them: (one bits, counts
        of the 256 byte values) -- the fused histogram consumer."""
        out = np.zeros(257, np.uint64)
        check(lib.vmt_stat_counts(self._h, n, out.ctypes.data, stream))
        return int(out[0]), out[1:].copy()

    def profile_totals(self) -> tuple[int, float, float]:
        """(fills, positioning-jump ms, generation ms) summed over the fills
        since profiling was enabled / the previous call; resets the sums."""
        n, j, gm = ctypes.c_uint64(), ctypes.c_double(), ctypes.c_double()
        check(lib.vmt_profile_totals(self._h, ctypes.byref(n), ctypes.byref(j), ctypes.byref(gm)))
        return n.value, j.value, gm.value

    def stats(self) -> dict:
        vals = [ctypes.c_uint64() for _ in range(4)]
        check(lib.vmt_stats(self._h, *[ctypes.byref(v) for v in vals]))
        return dict(zip(("gen_launches", "jump_launches", "other_launches", "lane_jumps"),
                        (v.value for v in vals)))


def VmtEngine(lanes: int, seed: int, jump_exponent: Optional[int] = None, device: int = 0) -> VmtGenerator:
    """VmtEngine<M>(seed, F^(2^q), q) (engine.hpp:54); M=1 needs no jump."""
    return VmtGenerator(seed, VmtConfig(lanes, QueryMode.kSingle, jump_exponent if lanes > 1 else 0), device)


def batch_fill_u32(out, seed0: int, ngen: int, lanes: int, n_per_gen: int,
                   jump_exponent: Optional[int] = None, device: int = 0, stream=None):
    """ngen generators seeded seed0.. (config 3): out[g*n_per_gen + i]."""
    addr, keep, size, kind = _ptr(out)
    _check_dtype(out, np.uint32, "uint32")
    if size < ngen * n_per_gen:
        raise InvalidArgument(_capi.VMT_EINVAL, "buffer too small")
    q = VMT_FULL_PERIOD if jump_exponent is None else jump_exponent
    check(lib.vmt_batch_fill_u32(seed0, ngen, lanes, q, n_per_gen, addr, device, _stream_for(kind, stream)))
    return out


class VmtBatch:
    """ngen independent generators (seeds seed0.., same lanes and de-phasing)
    advancing in lockstep (config 3); fill() continues every stream."""

    def __init__(self, seed0: int, ngen: int, lanes: int, jump_exponent: Optional[int] = None, device: int = 0):
        q = VMT_FULL_PERIOD if jump_exponent is None else jump_exponent
        self._h = ctypes.c_void_p()
        check(lib.vmt_batch_create(seed0 & 0xFFFFFFFF, ngen, lanes, q, device, ctypes.byref(self._h)))
        self.ngen, self.lanes, self.device = ngen, lanes, device

    def close(self) -> None:
        if self._h:
            check(lib.vmt_batch_destroy(self._h))
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def position(self) -> int:
        return int(lib.vmt_batch_position(self._h))

    def fill(self, out, n_per_gen: int, stream=None):
        _check_dtype(out, np.uint32, "uint32")
        addr, keep, size, kind = _ptr(out)
        if size < n_per_gen * self.ngen:
            raise InvalidArgument(_capi.VMT_EINVAL, "buffer smaller than ngen * n_per_gen")
        check(lib.vmt_batch_fill(self._h, addr, n_per_gen, _stream_for(kind, stream)))
        return out

    def skip(self, d: int) -> None:
        check(lib.vmt_batch_skip(self._h, d))

    def interleaved_states(self) -> np.ndarray:
        out = np.empty((self.ngen, KSTATE_LEN * self.lanes), np.uint32)
        check(lib.vmt_batch_export_state(self._h, out.ctypes.data))
        return out


def release_caches(device: int = 0) -> None:
    """Frees the process-wide de-phasing matrix cache of a device."""
    check(lib.vmt_release_caches(device))


def store_bandwidth(bytes_: int = 1 << 34, pattern: int = 0, ctas_per_sm: int = 2, device: int = 0) -> float:
    """GB/s of a pure-store probe kernel (0 grid-stride, 1 chunk per CTA, 2 chunk
    per CTA with random-looking words)."""
    out = ctypes.c_double()
    check(lib.vmt_store_bandwidth(device, bytes_, pattern, ctas_per_sm, ctypes.byref(out)))
    return out.value


def multi_gpu_fill(seed: int, lanes: int, n: int, devices, outs=None, jump_exponent: Optional[int] = None,
                   checksum: bool = True) -> Optional[int]:
    """vmt_multi_gpu_fill: words [0, n) of one stream split over `devices`
    (store into outs[k] on device k, or XOR only when outs is None)."""
    q = VMT_FULL_PERIOD if jump_exponent is None else jump_exponent
    devs = (ctypes.c_int * len(devices))(*devices)
    ptrs = None
    if outs is not None:
        ptrs = (ctypes.c_void_p * len(outs))(*[_ptr(o)[0] for o in outs])
    x = ctypes.c_uint32()
    check(lib.vmt_multi_gpu_fill(seed & 0xFFFFFFFF, lanes, q, n, len(devices), devs, ptrs,
                                 0 if outs is not None else 1, ctypes.byref(x) if checksum else None))
    return x.value if checksum else None


def jump_states(states, distances, out=None, device: int = 0, stream=None):
    """Advance n boundary states (n x 624, lane-major) by 64-bit distances (config 5)."""
    st = states
    if isinstance(states, np.ndarray):
        st = np.ascontiguousarray(states, np.uint32)
    saddr, _, ssize, kind = _ptr(st)
    n = ssize // KSTATE_LEN
    d = np.ascontiguousarray(distances, np.uint64)
    if d.size != n:
        raise InvalidArgument(_capi.VMT_EINVAL, "one distance per state")
    if out is None:
        out = np.empty((n, KSTATE_LEN), np.uint32) if kind == "cpu" else st.new_empty(st.shape)
    oaddr, _, _, _ = _ptr(out)
    check(lib.vmt_jump_states(saddr, n, d.ctypes.data, oaddr, device, _stream_for(kind, stream)))
    return out


def seed_states(seeds, device: int = 0) -> np.ndarray:
    s = np.ascontiguousarray(seeds, np.uint32)
    out = np.empty((s.size, KSTATE_LEN), np.uint32)
    check(lib.vmt_seed_states(s.ctypes.data, s.size, out.ctypes.data, device, None))
    return out


def charpoly() -> np.ndarray:
    out = np.empty(313, np.uint64)
    check(lib.vmt_charpoly(out.ctypes.data))
    return out


def jump_poly(d: int) -> np.ndarray:
    out = np.empty(312, np.uint64)
    check(lib.vmt_jump_poly(d & 0xFFFFFFFFFFFFFFFF, d >> 64, out.ctypes.data))
    return out


def jump_poly_pow2(q: int) -> np.ndarray:
    out = np.empty(312, np.uint64)
    check(lib.vmt_jump_poly_pow2(q, out.ctypes.data))
    return out


# ---- GF(2) jump matrices (f2_matrix.hpp, jump_file.hpp) ----------------------
def _matrix_out(out, device: int):
    if out is None:
        return np.empty((MATRIX_DIM, MATRIX_ROW_WORDS), np.uint64)
    _check_dtype(out, np.uint64, "uint64")
    if _ptr(out)[2] != MATRIX_WORDS:
        raise InvalidArgument(_capi.VMT_EINVAL, f"matrix buffer must have {MATRIX_WORDS} words")
    return out


def jump_matrix(d: int, out=None, device: int = 0, stream=None):
    """F^d (19937 x 312 uint64 rows; numpy by default, or a given numpy/torch
    buffer), computed on the GPU as 19937 polynomial jumps of basis states."""
    out = _matrix_out(out, device)
    addr, keep, _, kind = _ptr(out)
    check(lib.vmt_jump_matrix(d & (2**64 - 1), d >> 64, addr, device, _stream_for(kind, stream)))
    return out


def jump_matrix_pow2(q: int, out=None, device: int = 0, stream=None):
    """F^(2^q) == mat_pow2(build_transition_matrix(), q) (f2_matrix.cpp:138-228)."""
    out = _matrix_out(out, device)
    addr, keep, _, kind = _ptr(out)
    check(lib.vmt_jump_matrix_pow2(q, addr, device, _stream_for(kind, stream)))
    return out


def jump_matrix_file_name(exponent: int) -> str:
    """jump_file.cpp:167-169."""
    return f"F_2p{exponent}.vmtj"


def write_jump_matrix_file(path: str, rows, exponent: int) -> None:
    """write_jump_matrix_file (jump_file.cpp:117-123)."""
    addr, keep, n, _ = _ptr(rows)
    if n != MATRIX_WORDS:
        raise InvalidArgument(_capi.VMT_EINVAL, f"matrix must have {MATRIX_WORDS} uint64 words")
    check(lib.vmt_write_jump_matrix_file(str(path).encode(), addr, exponent))


def read_jump_matrix_file(path: str, rows: bool = True):
    """read_jump_matrix_file (jump_file.cpp:125-137): (rows or None, exponent).
    Format errors raise VmtError(VMT_EIO) like the reference's runtime_error."""
    e = ctypes.c_uint()
    if not rows:
        check(lib.vmt_read_jump_matrix_file(str(path).encode(), None, ctypes.byref(e)))
        return None, e.value
    out = np.empty((MATRIX_DIM, MATRIX_ROW_WORDS), np.uint64)
    check(lib.vmt_read_jump_matrix_file(str(path).encode(), out.ctypes.data, ctypes.byref(e)))
    return out, e.value


def compute_jump_matrix(exponent: int, out: str, device: int = 0) -> None:
    """compute_jump_matrix (jump_file.cpp:171-209): writes F^(2^exponent) to `out`."""
    check(lib.vmt_compute_jump_matrix_file(str(out).encode(), exponent, device))


def vec_mat_mul(vecs, rows, device: int = 0):
    """vec_mat_mul (f2_matrix.cpp:119-136) for n x 312 uint64 effective vectors."""
    v = np.ascontiguousarray(vecs, np.uint64).reshape(-1, MATRIX_ROW_WORDS)
    out = np.empty_like(v)
    addr, keep, n, _ = _ptr(rows)
    if n != MATRIX_WORDS:
        raise InvalidArgument(_capi.VMT_EINVAL, f"matrix must have {MATRIX_WORDS} uint64 words")
    check(lib.vmt_vec_mat_mul(v.ctypes.data, v.shape[0], addr, out.ctypes.data, device, None))
    return out


def jump_state_matrix(states, rows, device: int = 0):
    """jump_state (jump.cpp:27-33) with a caller matrix, n x 624 boundary states."""
    s = np.ascontiguousarray(states, np.uint32).reshape(-1, KSTATE_LEN)
    out = np.empty_like(s)
    addr, keep, n, _ = _ptr(rows)
    if n != MATRIX_WORDS:
        raise InvalidArgument(_capi.VMT_EINVAL, f"matrix must have {MATRIX_WORDS} uint64 words")
    check(lib.vmt_jump_states_matrix(s.ctypes.data, s.shape[0], addr, out.ctypes.data, device, None))
    return out


# ---- statistical smoke tests (stats.hpp) ---------------------------------------
K_SIGNIFICANCE = 0.001  # stats.hpp:24


class StatReport:
    """stats.hpp:13-20."""

    def __init__(self, name: str, samples: int, statistic: float, p_value: float, passed: bool):
        self.name, self.samples, self.statistic, self.p_value = name, samples, statistic, p_value
        self.pass_ = passed

    def __repr__(self) -> str:
        return (f"StatReport({self.name}, samples={self.samples}, statistic={self.statistic!r}, "
                f"p={self.p_value!r}, {'PASS' if self.pass_ else 'FAIL'})")


def _report(fn, gen: "VmtGenerator", count: int) -> StatReport:
    r = _capi.StatReportC()
    check(fn(gen._h, count, ctypes.byref(r)))
    return StatReport(r.name.decode(), r.samples, r.statistic, r.p_value, bool(r.pass_))


def monobit(gen: "VmtGenerator", count: int) -> StatReport:
    """monobit (stats.cpp:65-81) over the next `count` words of gen."""
    return _report(lib.vmt_monobit, gen, count)


def chi2_bytes(gen: "VmtGenerator", count: int) -> StatReport:
    """chi2_bytes (stats.cpp:83-107) over the next `count` words of gen."""
    return _report(lib.vmt_chi2_bytes, gen, count)


def lane_cross_correlation(gen: "VmtGenerator", count: int) -> StatReport:
    """lane_cross_correlation (stats.cpp:109-150) over the next count*lanes words."""
    return _report(lib.vmt_lane_cross_correlation, gen, count)


def monobit_from_counts(count: int, ones: int) -> StatReport:
    r = _capi.StatReportC()
    check(lib.vmt_monobit_from_counts(count, ones, ctypes.byref(r)))
    return StatReport(r.name.decode(), r.samples, r.statistic, r.p_value, bool(r.pass_))


def chi2_bytes_from_counts(count: int, bins) -> StatReport:
    b = np.ascontiguousarray(bins, np.uint64)
    if b.size != 256:
        raise InvalidArgument(_capi.VMT_EINVAL, "256 byte-value counts expected")
    r = _capi.StatReportC()
    check(lib.vmt_chi2_bytes_from_counts(count, b.ctypes.data, ctypes.byref(r)))
    return StatReport(r.name.decode(), r.samples, r.statistic, r.p_value, bool(r.pass_))


def stat_counts(gen: "VmtGenerator", n: int) -> tuple[int, np.ndarray]:
    return gen.stat_counts(n)


def regularized_gamma_q(a: float, x: float) -> float:
    """detail::regularized_gamma_q (stats.cpp:52-60)."""
    out = ctypes.c_double()
    check(lib.vmt_regularized_gamma_q(a, x, ctypes.byref(out)))
    return out.value
