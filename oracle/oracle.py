"""TEST INFRASTRUCTURE ONLY -- ctypes front end for the parity checkers.

* ``Oracle``  wraps ``oracle/liboracle.so``: the plain-C restatement of the
  reference algorithms (``oracle/vmt_oracle.c``; each function there cites the
  reference file:line it follows).
* ``RefLib``  wraps ``oracle/_ref/libvmtref.so``: the UNMODIFIED reference
  library (``/root/reference/proj/src``) behind a C shim (``oracle/ref_shim.cpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` (as the checker) and ``bench.py``'s
CPU arms may import this module. The product package never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from functools import lru_cache

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
DIM = 19937
RW = 312  # u64 words per 19937-bit vector (F2Vector::word_count)
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")


def build(quiet: bool = True) -> None:
    """Compile the oracle (and, when /root/reference is present, oracle/_ref)."""
    out = subprocess.run(["make", "-C", HERE, "all"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


class Oracle:
    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        lib = ctypes.CDLL(path)
        c = ctypes
        lib.or_temper.restype = c.c_uint32
        lib.or_temper.argtypes = [c.c_uint32]
        lib.or_mul_a.restype = c.c_uint32
        lib.or_mul_a.argtypes = [c.c_uint32]
        lib.or_seed.argtypes = [c.c_uint32, _u32p]
        lib.or_regenerate.argtypes = [_u32p]
        lib.or_mt_stream.argtypes = [c.c_uint32, c.c_uint64, c.c_uint64, _u32p]
        lib.or_mt_stream_from_words.argtypes = [_u32p, c.c_uint64, c.c_uint64, _u32p]
        lib.or_vmt_stream.argtypes = [_u32p, c.c_uint, c.c_uint64, c.c_uint64, _u32p]
        lib.or_vmt_checksum.restype = c.c_uint32
        lib.or_vmt_checksum.argtypes = [_u32p, c.c_uint, c.c_uint64, c.c_uint64]
        lib.or_vmt_regenerate.argtypes = [_u32p, c.c_uint]
        lib.or_words_to_effective.argtypes = [_u32p, _u64p]
        lib.or_effective_to_words.argtypes = [_u64p, _u32p]
        lib.or_build_transition.argtypes = [_u64p]
        lib.or_vec_mat_mul.argtypes = [_u64p, _u64p, _u64p]
        lib.or_mat_mul.argtypes = [_u64p, _u64p, _u64p]
        lib.or_jump_state_matrix.argtypes = [_u32p, _u64p, _u32p]
        lib.or_charpoly.restype = c.c_int
        lib.or_charpoly.argtypes = [_u64p]
        lib.or_poly_mulmod.argtypes = [_u64p, _u64p, _u64p, _u64p]
        lib.or_poly_sqrmod.argtypes = [_u64p, _u64p, _u64p]
        lib.or_x_pow_mod.argtypes = [c.c_uint64, _u64p, _u64p]
        lib.or_x_pow2_mod.argtypes = [c.c_uint, _u64p, _u64p]
        lib.or_poly_jump.argtypes = [_u32p, _u64p, _u32p]
        lib.or_mt64.argtypes = [c.c_uint64, c.c_uint64, _u64p]
        self.lib = lib

    # --- scalar core ---------------------------------------------------
    def temper(self, x: int) -> int:
        return self.lib.or_temper(x)

    def mul_a(self, u: int) -> int:
        return self.lib.or_mul_a(u)

    def seed_words(self, seed: int) -> np.ndarray:
        w = np.empty(624, np.uint32)
        self.lib.or_seed(seed, w)
        return w

    def mt_stream(self, seed: int, count: int, skip: int = 0) -> np.ndarray:
        out = np.empty(count, np.uint32)
        self.lib.or_mt_stream(seed, skip, count, out)
        return out

    def mt_stream_from_words(self, words: np.ndarray, count: int, skip: int = 0) -> np.ndarray:
        out = np.empty(count, np.uint32)
        self.lib.or_mt_stream_from_words(np.ascontiguousarray(words, np.uint32), skip, count, out)
        return out

    def mt64(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, np.uint64)
        self.lib.or_mt64(seed, count, out)
        return out

    # --- VMT engine ----------------------------------------------------
    def vmt_stream(self, lane_states: np.ndarray, start: int, count: int) -> np.ndarray:
        ls = np.ascontiguousarray(lane_states, np.uint32).reshape(-1)
        lanes = ls.size // 624
        out = np.empty(count, np.uint32)
        if self.lib.or_vmt_stream(ls, lanes, start, count, out) != 0:
            raise MemoryError
        return out

    def vmt_checksum(self, lane_states: np.ndarray, start: int, count: int) -> int:
        ls = np.ascontiguousarray(lane_states, np.uint32).reshape(-1)
        return int(self.lib.or_vmt_checksum(ls, ls.size // 624, start, count))

    # --- GF(2) ------------------------------------------------------------
    def transition_matrix(self) -> np.ndarray:
        f = np.empty(DIM * RW, np.uint64)
        self.lib.or_build_transition(f)
        return f

    def mat_mul(self, a: np.ndarray, b: np.ndarray) -> np.ndarray:
        c = np.empty_like(a)
        self.lib.or_mat_mul(a, b, c)
        return c

    def jump_state_matrix(self, words: np.ndarray, m: np.ndarray) -> np.ndarray:
        out = np.empty(624, np.uint32)
        self.lib.or_jump_state_matrix(np.ascontiguousarray(words, np.uint32), m, out)
        return out

    @lru_cache(maxsize=1)
    def charpoly(self) -> np.ndarray:
        p = np.zeros(313, np.uint64)
        deg = self.lib.or_charpoly(p)
        if deg != DIM:
            raise RuntimeError(f"Berlekamp-Massey returned degree {deg}")
        return p

    def x_pow_mod(self, d: int) -> np.ndarray:
        out = np.empty(RW, np.uint64)
        self.lib.or_x_pow_mod(d, self.charpoly(), out)
        return out

    def x_pow2_mod(self, q: int) -> np.ndarray:
        out = np.empty(RW, np.uint64)
        self.lib.or_x_pow2_mod(q, self.charpoly(), out)
        return out

    def mulmod(self, a: np.ndarray, b: np.ndarray) -> np.ndarray:
        out = np.empty(RW, np.uint64)
        self.lib.or_poly_mulmod(np.ascontiguousarray(a, np.uint64), np.ascontiguousarray(b, np.uint64),
                                self.charpoly(), out)
        return out

    def poly_pow(self, base: np.ndarray, e: int) -> np.ndarray:
        r = np.zeros(RW, np.uint64)
        r[0] = 1
        b = np.array(base, np.uint64)
        while e:
            if e & 1:
                r = self.mulmod(r, b)
            e >>= 1
            if e:
                b = self.mulmod(b, b)
        return r

    def poly_jump(self, words: np.ndarray, poly: np.ndarray) -> np.ndarray:
        out = np.empty(624, np.uint32)
        self.lib.or_poly_jump(np.ascontiguousarray(words, np.uint32),
                              np.ascontiguousarray(poly, np.uint64), out)
        return out

    def dephased_states(self, seed: int, lanes: int, base_poly: np.ndarray) -> np.ndarray:
        """Lane t = seed state jumped by t * 2^q, with base_poly = x^(2^q) mod P
        (make_dephased_states, jump.cpp:35-53, with the polynomial jump)."""
        st = np.empty((lanes, 624), np.uint32)
        st[0] = self.seed_words(seed)
        for t in range(1, lanes):
            st[t] = self.poly_jump(st[t - 1], base_poly)
        return st


class RefLib:
    """The unmodified reference library (oracle/_ref/libvmtref.so)."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "_ref", "libvmtref.so")
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        lib = ctypes.CDLL(path)
        c = ctypes
        lib.vref_mt_stream.argtypes = [c.c_uint32, c.c_uint64, c.c_uint64, _u32p]
        lib.vref_mt_stream_from_words.argtypes = [_u32p, c.c_uint64, _u32p]
        lib.vref_engine_stream.argtypes = [c.c_uint32, c.c_uint, c.c_uint, c.c_uint64, _u32p]
        lib.vref_engine_state.argtypes = [c.c_uint32, c.c_uint, c.c_uint, c.c_uint, _u32p]
        lib.vref_dephased_states.argtypes = [c.c_uint32, c.c_uint, c.c_uint, _u32p]
        lib.vref_jump_state.argtypes = [_u32p, c.c_uint, _u32p]
        lib.vref_seed_words.argtypes = [c.c_uint32, _u32p]
        lib.vref_prepare_ladder.argtypes = [c.c_uint]
        lib.vref_run_benchmark.argtypes = [c.c_uint, c.c_int, c.c_uint64, c.c_uint32, c.c_uint,
                                           c.POINTER(c.c_double), c.POINTER(c.c_uint32)]
        lib.vref_bench_threads.restype = c.c_double
        lib.vref_bench_threads.argtypes = [c.c_uint, c.c_uint32, c.c_uint, c.c_uint64, c.c_int,
                                           _u32p, c.POINTER(c.c_uint32)]
        lib.vref_simd_backend.argtypes = [c.c_uint]
        lib.vref_jump_by.argtypes = [_u32p, c.c_uint64, _u32p]
        lib.vref_mt64.argtypes = [c.c_uint64, c.c_uint64, _u64p]
        lib.vref_write_pow2_matrix_file.argtypes = [c.c_uint, c.c_char_p]
        lib.vref_read_jump_matrix_file.argtypes = [c.c_char_p, c.c_void_p, c.POINTER(c.c_uint),
                                                   c.POINTER(c.c_uint)]
        lib.vref_dephased_states_file.argtypes = [c.c_uint32, c.c_uint, c.c_char_p, _u32p]
        lib.vref_regularized_gamma_q.argtypes = [c.c_double, c.c_double, c.POINTER(c.c_double)]
        lib.vref_stat_report.argtypes = [c.c_uint32, c.c_uint, c.c_uint, c.c_uint64, c.c_int,
                                         c.POINTER(c.c_double), c.POINTER(c.c_double), c.POINTER(c.c_int)]
        for name in ("vref_lane_corr",):
            getattr(lib, name).argtypes = [c.c_uint32, c.c_uint, c.c_uint, c.c_uint64, c.POINTER(c.c_double),
                                           c.POINTER(c.c_double), c.POINTER(c.c_int)]
        lib.vref_stat_constant.argtypes = [c.c_uint32, c.c_uint64, c.c_int, c.POINTER(c.c_double),
                                           c.POINTER(c.c_double), c.POINTER(c.c_int)]
        self.lib = lib

    @staticmethod
    def _ok(rc: int, what: str) -> None:
        if rc != 0:
            raise RuntimeError(f"reference {what} failed rc={rc}")

    def mt_stream(self, seed, count, skip=0):
        out = np.empty(count, np.uint32)
        self._ok(self.lib.vref_mt_stream(seed, skip, count, out), "mt_stream")
        return out

    def engine_stream(self, seed, lanes, q, count):
        out = np.empty(count, np.uint32)
        self._ok(self.lib.vref_engine_stream(seed, lanes, q, count, out), "engine_stream")
        return out

    def engine_state(self, seed, lanes, q, nblocks):
        out = np.empty(624 * lanes, np.uint32)
        self._ok(self.lib.vref_engine_state(seed, lanes, q, nblocks, out), "engine_state")
        return out

    def dephased_states(self, seed, lanes, q):
        out = np.empty(624 * lanes, np.uint32)
        self._ok(self.lib.vref_dephased_states(seed, lanes, q, out), "dephased_states")
        return out.reshape(lanes, 624)

    def jump_state(self, words, q):
        out = np.empty(624, np.uint32)
        self._ok(self.lib.vref_jump_state(np.ascontiguousarray(words, np.uint32), q, out), "jump_state")
        return out

    def seed_words(self, seed):
        out = np.empty(624, np.uint32)
        self._ok(self.lib.vref_seed_words(seed, out), "seed_words")
        return out

    def jump_by(self, words, d):
        out = np.empty(624, np.uint32)
        self._ok(self.lib.vref_jump_by(np.ascontiguousarray(words, np.uint32), d, out), "jump_by")
        return out

    def mt64(self, seed, count):
        out = np.empty(count, np.uint64)
        self.lib.vref_mt64(seed, count, out)
        return out

    def write_pow2_matrix_file(self, q, path):
        """write_jump_matrix_file(path, F^(2^q), q) -- compute_jump_matrix's bytes."""
        self._ok(self.lib.vref_write_pow2_matrix_file(q, os.fsencode(path)), "write_jump_matrix_file")

    def read_jump_matrix_file(self, path, rows=True):
        """read_jump_matrix_file: (rows (dim, ceil(dim/64)) uint64 or None, exponent); raises
        RuntimeError(rc) on the reference's exceptions (-1 invalid_argument, -3 runtime_error)."""
        dim, e = ctypes.c_uint(), ctypes.c_uint()
        rc = self.lib.vref_read_jump_matrix_file(os.fsencode(path), None, ctypes.byref(dim), ctypes.byref(e))
        if rc != 0:
            raise RuntimeError(f"reference read_jump_matrix_file failed rc={rc}")
        if not rows:
            return None, e.value
        out = np.empty((dim.value, (dim.value + 63) // 64), np.uint64)
        self._ok(self.lib.vref_read_jump_matrix_file(os.fsencode(path), out.ctypes.data, None, None),
                 "read_jump_matrix_file")
        return out, e.value

    def dephased_states_file(self, seed, lanes, path):
        out = np.empty(624 * lanes, np.uint32)
        self._ok(self.lib.vref_dephased_states_file(seed, lanes, os.fsencode(path), out), "dephased_states_file")
        return out.reshape(lanes, 624)

    def regularized_gamma_q(self, a, x):
        out = ctypes.c_double()
        self._ok(self.lib.vref_regularized_gamma_q(a, x, ctypes.byref(out)), "regularized_gamma_q")
        return out.value

    def stat_report(self, seed, lanes, q, count, which):
        """(statistic, p_value, pass) of monobit (which=0) / chi2_bytes (1)."""
        st, p, ok = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
        self._ok(self.lib.vref_stat_report(seed, lanes, q, count, which, ctypes.byref(st), ctypes.byref(p),
                                           ctypes.byref(ok)), "stat_report")
        return st.value, p.value, bool(ok.value)

    def lane_corr(self, seed, lanes, q, count):
        st, p, ok = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
        self._ok(self.lib.vref_lane_corr(seed, lanes, q, count, ctypes.byref(st), ctypes.byref(p), ctypes.byref(ok)),
                 "lane_corr")
        return st.value, p.value, bool(ok.value)

    def stat_constant(self, word, count, which):
        st, p, ok = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
        self._ok(self.lib.vref_stat_constant(word, count, which, ctypes.byref(st), ctypes.byref(p),
                                             ctypes.byref(ok)), "stat_constant")
        return st.value, p.value, bool(ok.value)

    def run_benchmark(self, lanes, mode, count, seed, q):
        s = ctypes.c_double()
        x = ctypes.c_uint32()
        self._ok(self.lib.vref_run_benchmark(lanes, mode, count, seed, q, ctypes.byref(s), ctypes.byref(x)),
                 "run_benchmark")
        return s.value, x.value

    def bench_threads(self, lanes, seed, q, words_per_thread, threads, buf):
        x = ctypes.c_uint32()
        s = self.lib.vref_bench_threads(lanes, seed, q, words_per_thread, threads, buf, ctypes.byref(x))
        if s < 0:
            raise RuntimeError(f"reference bench_threads failed rc={s}")
        return s, x.value


def poly_bits_to_u64(bits: np.ndarray) -> np.ndarray:
    return np.packbits(bits.astype(np.uint8), bitorder="little").view(np.uint64)
