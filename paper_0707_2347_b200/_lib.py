"""ctypes binding of the C-ABI (include/winomem_b200.h).

Loads the in-tree ``libwinomem_b200.so``; there is no fallback -- if the library
is missing the import fails loudly (build it with ``python -m
paper_0707_2347_b200.build``).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
PRODUCT_LIB = os.path.join(HERE, "libwinomem_b200.so")
# the same library plus the measurement-only wm_diag_* probes (build.py); the
# measurement scripts select it with WM_DIAG=1, the product never does
DIAG_LIB = os.path.join(HERE, "libwinomem_b200_diag.so")
LIB_PATH = DIAG_LIB if os.environ.get("WM_DIAG") == "1" else PRODUCT_LIB

# status codes (winomem_b200.h)
WM_OK = 0
WM_FIELD_MODP = 0
WM_FIELD_REAL64 = 1

EXPORTS = [
    "wm_version", "wm_last_error", "wm_ctx_create", "wm_ctx_destroy", "wm_ctx_sync",
    "wm_ctx_set_option", "wm_ctx_get_option", "wm_block_addsub", "wm_block_scale_copy",
    "wm_classical_mul", "wm_run_variant", "wm_ipmm", "wm_run_variant_real",
    "wm_run_variant_host_u32", "wm_plan_report", "wm_expected_costs", "wm_plan_schedule_calls",
    "wm_plan_alloc_log",
    "wm_upload_u32", "wm_download_u32", "wm_fnv1a64_u32", "wm_fill_random",
    "wm_run_parsed_schedule", "wm_parse_schedule", "wm_render_schedule",
    "wm_run_parsed_schedule_host_u32", "wm_matrix_file_info", "wm_matrix_read_host",
    "wm_matrix_write_host", "wm_matrix_read_device", "wm_matrix_write_device",
    "wm_plan_report_parsed", "wm_lincomb", "wm_dev_alloc", "wm_dev_free", "wm_ctx_info",
    "wm_ctx_set_stream", "wm_dist_unique_id", "wm_dist_create", "wm_dist_destroy",
    "wm_dist_choose_levels", "wm_dist_run_variant", "wm_dist_last_error",
]


class wm_dmat(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("rows", C.c_uint64), ("cols", C.c_uint64),
                ("ld", C.c_uint64)]


class wm_dist_report(C.Structure):
    _fields_ = [("levels", C.c_int), ("products", C.c_uint64), ("peak_extra_bytes", C.c_uint64),
                ("bytes_sent", C.c_uint64), ("bytes_received", C.c_uint64)]


class wm_report(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "mults", "adds", "peak_extra_words", "total_alloc_words", "word_moves",
        "classical_calls", "schedule_frames", "peak_extra_bytes", "n_ops", "n_launches",
        "fused_frames", "add_bytes", "leaf_flops", "add_bytes_issued", "frame_gemm_bytes",
        "frame_bytes", "frame_prep_bytes", "frame_comb_bytes", "frame_leaf_flops")]


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the winomem-b200 native library must be built "
            "(python -m paper_0707_2347_b200.build); there is no fallback path")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    u32, u64, i32 = C.c_uint32, C.c_uint64, C.c_int
    ctx_p = C.c_void_p
    L.wm_version.restype = C.c_char_p
    L.wm_last_error.restype = C.c_char_p
    L.wm_ctx_create.argtypes = [i32, u32, i32, C.c_void_p, P(ctx_p)]
    L.wm_ctx_destroy.argtypes = [ctx_p]
    L.wm_ctx_sync.argtypes = [ctx_p]
    L.wm_ctx_set_option.argtypes = [ctx_p, C.c_char_p, C.c_int64]
    L.wm_ctx_get_option.argtypes = [ctx_p, C.c_char_p, P(C.c_int64)]
    L.wm_block_addsub.argtypes = [ctx_p, wm_dmat, wm_dmat, wm_dmat, u32, u32]
    L.wm_block_scale_copy.argtypes = [ctx_p, wm_dmat, wm_dmat, u32]
    L.wm_classical_mul.argtypes = [ctx_p, wm_dmat, wm_dmat, wm_dmat, u32, u32]
    L.wm_lincomb.argtypes = [ctx_p, wm_dmat, i32, P(wm_dmat), P(u32)]
    L.wm_run_variant.argtypes = [ctx_p, C.c_char_p, wm_dmat, wm_dmat, wm_dmat, u32, u32, i32,
                                 P(wm_report)]
    L.wm_ipmm.argtypes = [ctx_p, wm_dmat, wm_dmat, wm_dmat, i32, P(wm_report)]
    L.wm_run_variant_real.argtypes = [ctx_p, C.c_char_p, wm_dmat, wm_dmat, wm_dmat, C.c_double,
                                      C.c_double, i32, P(wm_report)]
    L.wm_run_variant_host_u32.argtypes = [ctx_p, C.c_char_p, u64, u64, u64, C.c_void_p,
                                          C.c_void_p, C.c_void_p, u32, u32, i32, P(wm_report)]
    L.wm_plan_report.argtypes = [C.c_char_p, i32, u32, u64, u64, u64, u32, u32, i32, i32,
                                 P(wm_report)]
    L.wm_expected_costs.argtypes = [C.c_char_p, u64, u64, u64, i32, P(wm_report)]
    L.wm_plan_schedule_calls.argtypes = [C.c_char_p, i32]
    L.wm_plan_alloc_log.argtypes = [C.c_char_p, i32]
    L.wm_upload_u32.argtypes = [ctx_p, wm_dmat, C.c_void_p, u64]
    L.wm_download_u32.argtypes = [ctx_p, C.c_void_p, u64, wm_dmat]
    L.wm_fnv1a64_u32.argtypes = [C.c_void_p, u64]
    L.wm_fnv1a64_u32.restype = u64
    L.wm_fill_random.argtypes = [ctx_p, wm_dmat, u64]
    L.wm_run_parsed_schedule.argtypes = [ctx_p, C.c_char_p, wm_dmat, wm_dmat, wm_dmat, u32, u32,
                                         i32, P(wm_report)]
    L.wm_parse_schedule.argtypes = [C.c_char_p, C.c_char_p, i32, P(i32), P(i32)]
    L.wm_render_schedule.argtypes = [C.c_char_p, C.c_char_p, i32, P(i32)]
    L.wm_plan_report_parsed.argtypes = [C.c_char_p, u32, u64, u64, u64, u32, u32, i32, P(wm_report)]
    L.wm_matrix_file_info.argtypes = [C.c_char_p, i32, P(u64), P(u64), P(u32)]
    L.wm_matrix_read_host.argtypes = [C.c_char_p, i32, C.c_void_p, u64]
    L.wm_matrix_write_host.argtypes = [C.c_char_p, i32, u64, u64, u32, C.c_void_p]
    L.wm_matrix_read_device.argtypes = [ctx_p, C.c_char_p, i32, wm_dmat]
    L.wm_matrix_write_device.argtypes = [ctx_p, C.c_char_p, i32, wm_dmat]
    L.wm_run_parsed_schedule_host_u32.argtypes = [ctx_p, C.c_char_p, u64, u64, u64, C.c_void_p,
                                                  C.c_void_p, C.c_void_p, u32, u32, i32,
                                                  P(wm_report)]
    L.wm_ctx_info.argtypes = [ctx_p, P(i32), P(u32), P(i32), P(C.c_void_p)]
    L.wm_ctx_set_stream.argtypes = [ctx_p, C.c_void_p]
    L.wm_dist_unique_id.argtypes = [C.c_char_p]
    L.wm_dist_create.argtypes = [ctx_p, i32, i32, C.c_char_p, P(C.c_void_p)]
    L.wm_dist_destroy.argtypes = [C.c_void_p]
    L.wm_dist_choose_levels.argtypes = [i32, u64, i32]
    L.wm_dist_run_variant.argtypes = [C.c_void_p, C.c_char_p, wm_dmat, wm_dmat, wm_dmat, u32, u32,
                                      i32, i32, i32, P(wm_dist_report)]
    L.wm_dist_last_error.restype = C.c_char_p
    _lib = L
    return L


_diag = None


def diag_lib():
    """The diagnostics library on its own (own contexts): kernel-level checks
    that need a wm_diag_* entry point without switching the product library."""
    global _diag
    if _diag is None:
        if not os.path.exists(DIAG_LIB):
            raise ImportError(f"{DIAG_LIB} is missing (python -m paper_0707_2347_b200.build)")
        L = C.CDLL(DIAG_LIB)
        L.wm_ctx_create.argtypes = [C.c_int, C.c_uint32, C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]
        L.wm_ctx_destroy.argtypes = [C.c_void_p]
        L.wm_last_error.restype = C.c_char_p
        _diag = L
    return _diag


def last_error():
    return lib().wm_last_error().decode(errors="replace")
