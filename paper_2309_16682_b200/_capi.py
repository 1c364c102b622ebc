"""ctypes binding of the C ABI in include/vmt19937_b200.h.

Loads the in-tree libvmt19937_b200.so. There is deliberately no fallback: if
the library is missing the import fails, and without a CUDA device every
generating call raises VmtError(VMT_ECUDA).
"""
from __future__ import annotations

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# VMT_LIB: A/B experiments only (another build of the same sources)
LIB_PATH = os.environ.get("VMT_LIB") or os.path.join(PKG, "libvmt19937_b200.so")

VMT_OK, VMT_EINVAL, VMT_ESTATE, VMT_EIO, VMT_ECUDA, VMT_ENOMEM = 0, -1, -2, -3, -4, -5
VMT_FULL_PERIOD = 0xFFFFFFFF
VMT_PREFETCH_OFF, VMT_PREFETCH_JUMPS, VMT_PREFETCH_TENSOR = 0, 1, 2
VMT_F32_24, VMT_F64_32, VMT_F64_REAL3, VMT_F64_RES53 = 0, 1, 2, 3

# every symbol include/vmt19937_b200.h declares
EXPORTS = [
    "vmt_full_period_exponent", "vmt_create", "vmt_create_from_states", "vmt_clone", "vmt_destroy", "vmt_lanes",
    "vmt_state_words", "vmt_jump_exponent", "vmt_position", "vmt_next_u32", "vmt_next_block16",
    "vmt_next_block_state", "vmt_fill_u32", "vmt_fill_f32", "vmt_fill_f64", "vmt_checksum_xor",
    "vmt_skip", "vmt_seek", "vmt_synchronize", "vmt_export_state", "vmt_batch_fill_u32", "vmt_jump_states", "vmt_seed_states",
    "vmt_jump_poly", "vmt_jump_poly_pow2", "vmt_charpoly", "vmt_set_tuning", "vmt_set_prefetch", "vmt_prefetch_stats", "vmt_set_profiling", "vmt_last_timings", "vmt_profile_totals", "vmt_stats",
    "vmt_status_string", "vmt_last_error", "vmt_version",
    "vmt_jump_matrix", "vmt_jump_matrix_pow2", "vmt_write_jump_matrix_file", "vmt_read_jump_matrix_file",
    "vmt_compute_jump_matrix_file", "vmt_vec_mat_mul", "vmt_jump_states_matrix", "vmt_create_from_matrix",
    "vmt_create_from_file", "vmt_stat_counts", "vmt_monobit", "vmt_chi2_bytes", "vmt_regularized_gamma_q",
    "vmt_monobit_from_counts", "vmt_chi2_bytes_from_counts", "vmt_lane_cross_correlation",
    "vmt_lane_cross_correlation_from_words",
    "vmt_batch_create", "vmt_batch_fill", "vmt_batch_skip", "vmt_batch_position", "vmt_batch_export_state",
    "vmt_batch_destroy", "vmt_multi_gpu_fill", "vmt_store_bandwidth",
    "vmt_set_positioning", "vmt_positioning_stats", "vmt_release_caches",
]


class StatReportC(ctypes.Structure):
    """vmt_stat_report (StatReport, stats.hpp:13-20)."""
    _fields_ = [("name", ctypes.c_char_p), ("samples", ctypes.c_uint64), ("statistic", ctypes.c_double),
                ("p_value", ctypes.c_double), ("pass_", ctypes.c_int)]


class VmtError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class InvalidArgument(VmtError, ValueError):
    """std::invalid_argument in the reference."""


class LogicError(VmtError):
    """std::logic_error in the reference (cadence / boundary)."""


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2309_16682_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    c = ctypes
    H = c.c_void_p
    u32p, u64p = c.POINTER(c.c_uint32), c.POINTER(c.c_uint64)
    sig = {
        "vmt_full_period_exponent": (c.c_uint, [c.c_uint]),
        "vmt_create": (c.c_int, [c.c_uint32, c.c_uint, c.c_uint, c.c_int, c.POINTER(H)]),
        "vmt_create_from_states": (c.c_int, [c.c_void_p, c.c_uint, c.c_int, c.POINTER(H)]),
        "vmt_destroy": (c.c_int, [H]),
        "vmt_lanes": (c.c_uint, [H]),
        "vmt_state_words": (c.c_uint64, [H]),
        "vmt_jump_exponent": (c.c_uint, [H]),
        "vmt_position": (c.c_uint64, [H]),
        "vmt_next_u32": (c.c_int, [H, u32p]),
        "vmt_next_block16": (c.c_int, [H, c.c_void_p]),
        "vmt_next_block_state": (c.c_int, [H, c.c_void_p]),
        "vmt_fill_u32": (c.c_int, [H, c.c_void_p, c.c_uint64, c.c_void_p]),
        "vmt_fill_f32": (c.c_int, [H, c.c_void_p, c.c_uint64, c.c_int, c.c_void_p]),
        "vmt_fill_f64": (c.c_int, [H, c.c_void_p, c.c_uint64, c.c_int, c.c_void_p]),
        "vmt_checksum_xor": (c.c_int, [H, c.c_uint64, u32p, c.c_void_p]),
        "vmt_skip": (c.c_int, [H, c.c_uint64]),
        "vmt_seek": (c.c_int, [H, c.c_uint64]),
        "vmt_synchronize": (c.c_int, [H]),
        "vmt_export_state": (c.c_int, [H, c.c_void_p]),
        "vmt_batch_fill_u32": (c.c_int, [c.c_uint32, c.c_uint, c.c_uint, c.c_uint, c.c_uint64, c.c_void_p,
                                         c.c_int, c.c_void_p]),
        "vmt_jump_states": (c.c_int, [c.c_void_p, c.c_uint64, c.c_void_p, c.c_void_p, c.c_int, c.c_void_p]),
        "vmt_seed_states": (c.c_int, [c.c_void_p, c.c_uint64, c.c_void_p, c.c_int, c.c_void_p]),
        "vmt_jump_poly": (c.c_int, [c.c_uint64, c.c_uint64, c.c_void_p]),
        "vmt_jump_poly_pow2": (c.c_int, [c.c_uint, c.c_void_p]),
        "vmt_charpoly": (c.c_int, [c.c_void_p]),
        "vmt_set_tuning": (c.c_int, [H, c.c_uint, c.c_int]),
        "vmt_set_prefetch": (c.c_int, [H, c.c_int]),
        "vmt_prefetch_stats": (c.c_int, [H, u64p, u64p]),
        "vmt_stats": (c.c_int, [H, u64p, u64p, u64p, u64p]),
        "vmt_set_profiling": (c.c_int, [H, c.c_int]),
        "vmt_last_timings": (c.c_int, [H, c.POINTER(c.c_float), c.POINTER(c.c_float)]),
        "vmt_profile_totals": (c.c_int, [H, u64p, c.POINTER(c.c_double), c.POINTER(c.c_double)]),
        "vmt_status_string": (c.c_char_p, [c.c_int]),
        "vmt_last_error": (c.c_char_p, []),
        "vmt_version": (c.c_int, []),
        "vmt_jump_matrix": (c.c_int, [c.c_uint64, c.c_uint64, c.c_void_p, c.c_int, c.c_void_p]),
        "vmt_jump_matrix_pow2": (c.c_int, [c.c_uint, c.c_void_p, c.c_int, c.c_void_p]),
        "vmt_write_jump_matrix_file": (c.c_int, [c.c_char_p, c.c_void_p, c.c_uint]),
        "vmt_read_jump_matrix_file": (c.c_int, [c.c_char_p, c.c_void_p, c.POINTER(c.c_uint)]),
        "vmt_compute_jump_matrix_file": (c.c_int, [c.c_char_p, c.c_uint, c.c_int]),
        "vmt_vec_mat_mul": (c.c_int, [c.c_void_p, c.c_uint64, c.c_void_p, c.c_void_p, c.c_int, c.c_void_p]),
        "vmt_jump_states_matrix": (c.c_int, [c.c_void_p, c.c_uint64, c.c_void_p, c.c_void_p, c.c_int,
                                             c.c_void_p]),
        "vmt_create_from_matrix": (c.c_int, [c.c_uint32, c.c_uint, c.c_void_p, c.c_uint, c.c_int, c.POINTER(H)]),
        "vmt_create_from_file": (c.c_int, [c.c_uint32, c.c_uint, c.c_char_p, c.c_int, c.POINTER(H)]),
        "vmt_stat_counts": (c.c_int, [H, c.c_uint64, c.c_void_p, c.c_void_p]),
        "vmt_monobit": (c.c_int, [H, c.c_uint64, c.POINTER(StatReportC)]),
        "vmt_chi2_bytes": (c.c_int, [H, c.c_uint64, c.POINTER(StatReportC)]),
        "vmt_regularized_gamma_q": (c.c_int, [c.c_double, c.c_double, c.POINTER(c.c_double)]),
        "vmt_monobit_from_counts": (c.c_int, [c.c_uint64, c.c_uint64, c.POINTER(StatReportC)]),
        "vmt_chi2_bytes_from_counts": (c.c_int, [c.c_uint64, c.c_void_p, c.POINTER(StatReportC)]),
        "vmt_lane_cross_correlation": (c.c_int, [H, c.c_uint64, c.POINTER(StatReportC)]),
        "vmt_batch_create": (c.c_int, [c.c_uint32, c.c_uint, c.c_uint, c.c_uint, c.c_int, c.POINTER(H)]),
        "vmt_batch_fill": (c.c_int, [H, c.c_void_p, c.c_uint64, c.c_void_p]),
        "vmt_batch_skip": (c.c_int, [H, c.c_uint64]),
        "vmt_batch_position": (c.c_uint64, [H]),
        "vmt_batch_export_state": (c.c_int, [H, c.c_void_p]),
        "vmt_batch_destroy": (c.c_int, [H]),
        "vmt_set_positioning": (c.c_int, [H, c.c_int]),
        "vmt_release_caches": (c.c_int, [c.c_int]),
        "vmt_positioning_stats": (c.c_int, [H, u64p, u64p]),
        "vmt_store_bandwidth": (c.c_int, [c.c_int, c.c_uint64, c.c_int, c.c_int, c.POINTER(c.c_double)]),
        "vmt_multi_gpu_fill": (c.c_int, [c.c_uint32, c.c_uint, c.c_uint, c.c_uint64, c.c_int,
                                         c.POINTER(c.c_int), c.POINTER(c.c_void_p), c.c_int, u32p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(rc: int) -> None:
    if rc == VMT_OK:
        return
    msg = (lib.vmt_last_error() or b"").decode(errors="replace")
    if rc == VMT_EINVAL:
        raise InvalidArgument(rc, msg)
    if rc == VMT_ESTATE:
        raise LogicError(rc, msg)
    raise VmtError(rc, msg)
