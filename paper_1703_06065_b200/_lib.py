"""ctypes binding of libbcur_b200.so (the C ABI declared in include/bcur_b200.h).

The library is built in-tree (``python -m paper_1703_06065_b200.build``).  There
is no fallback: if the shared object is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbcur_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing — build the sm_100a library first "
        "(python -m paper_1703_06065_b200.build); there is no CPU fallback")

lib = C.CDLL(LIB_PATH)

i64 = C.c_int64
u64 = C.c_uint64
dbl = C.c_double
vp = C.c_void_p
P_i64 = C.POINTER(i64)
P_dbl = C.POINTER(dbl)


class RowDrawC(C.Structure):
    _fields_ = [("row", C.c_int64), ("probability", C.c_double), ("scale", C.c_double)]


class Alg1ReportC(C.Structure):
    _fields_ = [("abs_err_u", C.c_double), ("abs_err_uk", C.c_double), ("a_norm", C.c_double),
                ("rank_r", C.c_int64), ("rank_w", C.c_int64)]


class BlockDrawC(C.Structure):
    _fields_ = [("block", i64), ("probability", dbl), ("scale", dbl)]


class OptionsC(C.Structure):
    _fields_ = [("k", i64), ("p", i64), ("q", i64), ("g", i64), ("g_rows", i64), ("mode", C.c_int),
                ("residual", C.c_int), ("seed", u64), ("rank_floor", C.c_int)]


class ReportC(C.Structure):
    _fields_ = [("abs_err", dbl), ("a_norm", dbl), ("rel_err", dbl), ("k_eff", i64), ("rank_c", i64),
                ("rank_r", i64), ("residual_path", C.c_int), ("orth_dev", dbl)]


class GreedyStepC(C.Structure):
    _fields_ = [("block", i64), ("score", dbl), ("margin", dbl), ("saturated", C.c_int), ("rank_added", i64)]


class GenSpecC(C.Structure):
    _fields_ = [("kind", C.c_int), ("dtype", C.c_int), ("m", i64), ("n", i64), ("rank", i64), ("sigma", P_dbl),
                ("noise", dbl), ("seed", u64), ("col0", i64), ("n_global", i64)]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, vp, P_dbl, i64, vp)
BROADCAST_FN = C.CFUNCTYPE(C.c_int, vp, vp, i64, C.c_int, vp)


class CommC(C.Structure):
    _fields_ = [("rank", C.c_int), ("world", C.c_int), ("user", vp), ("allreduce_f64", ALLREDUCE_FN),
                ("broadcast", BROADCAST_FN)]


# name: (restype, argtypes)
SIGNATURES = {
    "bcur_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "bcur_ctx_destroy": (C.c_int, [vp]),
    "bcur_ctx_set_stream": (C.c_int, [vp, vp]),
    "bcur_ctx_stream": (vp, [vp]),
    "bcur_ctx_synchronize": (C.c_int, [vp]),
    "bcur_ctx_launch_count": (i64, [vp]),
    "bcur_ctx_profile": (C.c_int, [vp, C.c_int]),
    "bcur_ctx_profile_dump": (i64, [vp, C.c_char_p, i64]),
    "bcur_ctx_set_comm": (C.c_int, [vp, C.POINTER(CommC)]),
    "bcur_dmat_create": (C.c_int, [vp, C.c_int, i64, i64, C.POINTER(vp)]),
    "bcur_dmat_upload": (C.c_int, [vp, vp, vp, i64]),
    "bcur_dmat_upload_async": (C.c_int, [vp, vp, vp, i64]),
    "bcur_bcur_header": (C.c_int, [C.c_char_p, C.POINTER(i64), C.POINTER(i64)]),
    "bcur_dmat_load_bcur": (C.c_int, [vp, C.c_char_p, C.c_int, i64, i64, C.POINTER(vp)]),
    "bcur_dmat_save_bcur": (C.c_int, [vp, vp, C.c_char_p]),
    "bcur_dmat_download": (C.c_int, [vp, vp, vp, i64]),
    "bcur_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(vp)]),
    "bcur_host_free": (C.c_int, [vp]),
    "bcur_dmat_wrap": (C.c_int, [vp, C.c_int, i64, i64, vp, i64, C.POINTER(vp)]),
    "bcur_dmat_info": (C.c_int, [vp, C.POINTER(C.c_int), P_i64, P_i64, P_i64, C.POINTER(vp)]),
    "bcur_dmat_set_shard": (C.c_int, [vp, i64, i64]),
    "bcur_dmat_destroy": (C.c_int, [vp]),
    "bcur_dmat_generate": (C.c_int, [vp, C.POINTER(GenSpecC), C.POINTER(vp)]),
    "bcur_rng_create": (C.c_int, [u64, C.POINTER(vp)]),
    "bcur_rng_destroy": (C.c_int, [vp]),
    "bcur_rng_seed": (u64, [vp]),
    "bcur_rng_next_u64": (u64, [vp]),
    "bcur_rng_uniform01": (dbl, [vp]),
    "bcur_rng_below": (u64, [vp, u64]),
    "bcur_rng_normal": (dbl, [vp]),
    "bcur_rng_split_seed": (u64, [vp, u64]),
    "bcur_omega_key": (u64, [u64]),
    "bcur_frobenius_norm": (C.c_int, [vp, vp, P_dbl]),
    "bcur_block_sq_norms": (C.c_int, [vp, vp, P_i64, i64, P_dbl]),
    "bcur_block_leverage": (C.c_int, [vp, vp, P_i64, i64, dbl, P_dbl, P_dbl]),
    "bcur_column_leverage": (C.c_int, [vp, vp, dbl, P_dbl, P_dbl]),
    "bcur_range_finder": (C.c_int, [vp, vp, i64, i64, i64, u64, C.POINTER(vp), C.POINTER(vp), P_dbl, P_i64]),
    "bcur_sketch_product": (C.c_int, [vp, vp, vp, C.c_int, vp, P_dbl]),
    "bcur_sketch_product_ex": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, vp]),
    "bcur_cholesky": (C.c_int, [vp, vp, vp, vp, C.POINTER(C.c_int), P_dbl]),
    "bcur_draw_blocks": (C.c_int, [vp, P_dbl, i64, i64, C.c_int, P_dbl, u64, C.POINTER(BlockDrawC), P_dbl]),
    "bcur_materialize_columns": (C.c_int, [vp, vp, P_i64, i64, C.POINTER(BlockDrawC), i64, C.POINTER(vp)]),
    "bcur_materialize_row_blocks": (C.c_int, [vp, vp, P_i64, i64, C.POINTER(BlockDrawC), i64, C.POINTER(vp)]),
    "bcur_error_report": (C.c_int, [vp, vp, vp, vp, vp, P_dbl, P_dbl]),
    "bcur_block_cur_alg1": (C.c_int, [vp, vp, P_i64, i64, i64, C.POINTER(RowDrawC), i64, C.c_int, i64, C.c_int,
                                      P_dbl, P_dbl, P_dbl, C.POINTER(BlockDrawC), P_dbl, P_dbl,
                                      C.POINTER(Alg1ReportC)]),
    "bcur_block_diagnostics": (C.c_int, [vp, vp, vp, P_i64, i64, P_dbl, P_dbl, P_dbl]),
    "bcur_block_css": (C.c_int, [vp, vp, P_i64, i64, C.POINTER(OptionsC), P_dbl, P_dbl, P_dbl,
                                 C.POINTER(BlockDrawC), P_dbl, C.POINTER(ReportC)]),
    "bcur_greedy_select": (C.c_int, [vp, vp, P_i64, i64, C.POINTER(OptionsC), C.POINTER(GreedyStepC), P_dbl,
                                     C.POINTER(ReportC)]),
    "bcur_block_cur": (C.c_int, [vp, vp, P_i64, i64, P_i64, i64, C.POINTER(OptionsC), P_dbl, P_dbl, P_dbl,
                                 C.POINTER(BlockDrawC), C.POINTER(BlockDrawC), P_dbl, i64, C.POINTER(ReportC)]),
    "bcur_last_error": (C.c_char_p, []),
    "bcur_version": (C.c_char_p, []),
}

for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

# status codes (bcur_status)
OK = 0
STATUS_NAMES = {
    1: "INVALID_ARGUMENT", 2: "OUT_OF_RANGE", 3: "DIMENSION_MISMATCH", 4: "INVALID_BASIS", 5: "ZERO_BLOCK",
    6: "ZERO_MATRIX", 7: "DISTRIBUTION_INVALID", 8: "NOT_ENOUGH_BLOCKS", 9: "DEGENERATE_R",
    10: "ITERATION_FAILURE", 11: "PARSE", 12: "CUDA", 13: "COMM",
}
F32, F64 = 0, 1
WITH_REPLACEMENT, WITHOUT_REPLACEMENT = 0, 1
RESID_AUTO, RESID_PYTHAGORAS, RESID_EXPLICIT = -1, 0, 1
GEN_LOWRANK, GEN_BIOMETRIC = 0, 1


def last_error() -> str:
    return lib.bcur_last_error().decode("utf-8", "replace")
