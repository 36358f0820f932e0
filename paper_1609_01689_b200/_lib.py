"""ctypes binding of libcieg.so (include/cieg.h).

The shared object is built in-tree by ``paper_1609_01689_b200/csrc/Makefile``
(``__graft_entry__.build()``). There is no fallback: if the library cannot be
loaded, every entry point raises ``ImportError`` -- the product path never
routes through the CPU oracle.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib

_HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = pathlib.Path(os.environ["CIEG_LIB"]) if os.environ.get("CIEG_LIB") else _HERE / "libcieg.so"  # override: experiments


class CsbView(C.Structure):
    _fields_ = [
        ("dim", C.c_uint32),
        ("nb", C.c_uint32),
        ("precision", C.c_int),
        ("block_boundaries", C.POINTER(C.c_uint32)),
        ("entry_offsets", C.POINTER(C.c_uint64)),
        ("rows", C.POINTER(C.c_uint16)),
        ("cols", C.POINTER(C.c_uint16)),
        ("values", C.c_void_p),
    ]


class GenParams(C.Structure):
    _fields_ = [
        ("n", C.c_uint32),
        ("sectors", C.c_uint32),
        ("tile", C.c_uint32),
        ("band", C.c_uint32),
        ("p", C.c_double),
        ("q", C.c_double),
        ("seed", C.c_uint64),
        ("precision", C.c_int),
        ("beta", C.c_uint32),
    ]


class PrecondConfigC(C.Structure):
    _fields_ = [
        ("inner_iters", C.c_int),
        ("small_block_cutoff", C.c_int),
        ("engage_after", C.c_int),
        ("relres_gate", C.c_double),
        ("near_converged_factor", C.c_double),
        ("far_threshold", C.c_double),
        ("column_floor_factor", C.c_double),
    ]


class TileDiagView(C.Structure):
    _fields_ = [
        ("dim", C.c_uint32),
        ("ngroups", C.c_uint32),
        ("bounds", C.POINTER(C.c_uint32)),
        ("blocks", C.POINTER(C.c_double)),
    ]


class LobpcgOptionsC(C.Structure):
    _fields_ = [
        ("k_want", C.c_int),
        ("tol", C.c_double),
        ("max_iter", C.c_int),
        ("precond_config", PrecondConfigC),
    ]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_uint64)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p)


PARTIALS_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p)


class DistHooks(C.Structure):
    _fields_ = [("user", C.c_void_p), ("allreduce_sum", ALLREDUCE_FN), ("allgather_rows", ALLGATHER_FN),
                ("reduce_partials", PARTIALS_FN)]


OBSERVER = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.POINTER(C.c_double), C.c_uint32,
                       C.c_uint32, C.POINTER(C.c_double), C.POINTER(C.c_double))

class MultilevelOptionsC(C.Structure):
    _fields_ = [
        ("k_want", C.c_int),
        ("k_trial", C.c_int),
        ("tol", C.c_double),
        ("max_iter", C.c_int),
        ("seed", C.c_uint64),
    ]


class LevelReportC(C.Structure):
    _fields_ = [
        ("dim", C.c_uint32),
        ("iterations", C.c_int),
        ("converged", C.c_int),
        ("seconds", C.c_double),
    ]


# cieg_lanczos_observer_fn(user, m, alpha, beta, basis_host (n x m col-major), n)
LANCZOS_OBSERVER = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                               C.POINTER(C.c_double), C.c_uint32)


class LanczosOptionsC(C.Structure):
    _fields_ = [
        ("k_want", C.c_int),
        ("tol", C.c_double),
        ("max_iter", C.c_int),
        ("observer", LANCZOS_OBSERVER),
        ("observer_user", C.c_void_p),
    ]

_vp = C.c_void_p
_u32 = C.c_uint32
_u64 = C.c_uint64
_i = C.c_int
_d = C.c_double
_pd = C.POINTER(C.c_double)
_pu32 = C.POINTER(C.c_uint32)
_pu64 = C.POINTER(C.c_uint64)
_pi = C.POINTER(C.c_int)

# name: (restype, argtypes)
SIGNATURES = {
    "cieg_last_error": (C.c_char_p, []),
    "cieg_version": (C.c_char_p, []),
    "cieg_ctx_create": (_i, [_i, C.POINTER(_vp)]),
    "cieg_ctx_destroy": (_i, [_vp]),
    "cieg_ctx_synchronize": (_i, [_vp]),
    "cieg_ctx_stream": (_vp, [_vp]),
    "cieg_ctx_launch_count": (_u64, [_vp]),
    "cieg_matrix_upload": (_i, [_vp, C.POINTER(CsbView), _pu32, _u32, _u32, C.POINTER(_vp)]),
    "cieg_matrix_destroy": (_i, [_vp]),
    "cieg_matrix_info": (_i, [_vp, _pu32, _pu64, _pu32, _pu64, _pu32, _pi, _pu64]),
    "cieg_spmm": (_i, [_vp, _vp, _vp, _vp, _u32]),
    "cieg_spmm_host": (_i, [_vp, _vp, _pd, _pd, _u32]),
    "cieg_block_inner": (_i, [_vp, _u32, _vp, _u32, _vp, _u32, _pd]),
    "cieg_linear_combination": (_i, [_vp, _u32, _vp, _u32, _pd, _u32, _vp]),
    "cieg_add_linear_combination": (_i, [_vp, _u32, _vp, _u32, _vp, _u32, _pd]),
    "cieg_column_norms": (_i, [_vp, _u32, _vp, _u32, _pd]),
    "cieg_precond_config_default": (None, [C.POINTER(PrecondConfigC)]),
    "cieg_precond_upload": (_i, [_vp, C.POINTER(TileDiagView), C.POINTER(_vp)]),
    "cieg_precond_from_csb": (_i, [_vp, C.POINTER(CsbView), _pu32, _u32, C.POINTER(_vp)]),
    "cieg_precond_destroy": (_i, [_vp]),
    "cieg_choose_shifts": (_i, [_u32, _pd, _pd, _pd, _pd, _i, _d, C.POINTER(PrecondConfigC), _pd, _pi]),
    "cieg_precond_apply": (_i, [_vp, _vp, _vp, _u32, _pd, _pi, C.POINTER(PrecondConfigC), _vp]),
    "cieg_lobpcg_options_default": (None, [C.POINTER(LobpcgOptionsC)]),
    "cieg_lobpcg_solve": (_i, [_vp, _vp, _pd, _u32, _vp, C.POINTER(LobpcgOptionsC), OBSERVER, _vp,
                               C.POINTER(_vp)]),
    "cieg_report_destroy": (_i, [_vp]),
    "cieg_lanczos_options_default": (None, [C.POINTER(LanczosOptionsC)]),
    "cieg_device_alloc": (_i, [_vp, C.c_uint64, C.POINTER(_vp)]),
    "cieg_random_block_rows": (_i, [_u32, _u32, _u32, C.c_uint64, _pd]),
    "cieg_spmm_host_batch": (_i, [_vp, _vp, C.POINTER(_pd), C.POINTER(_pd), _u32, _u32]),
    "cieg_device_free": (_i, [_vp, _vp]),
    "cieg_memcpy": (_i, [_vp, _vp, _vp, C.c_uint64, C.c_int]),
    "cieg_orthonormalize": (_i, [_vp, _vp, _u32, _u32, C.c_double, _vp, _u32, _pu32]),
    "cieg_rayleigh_ritz": (_i, [_vp, _vp, _vp, _u32, _u32, _u32, _pd, _pd]),
    "cieg_residual_norms": (_i, [_vp, _vp, _vp, _u32, _pd, C.c_double, _pd]),
    "cieg_matrix_leading_view": (_i, [_vp, _vp, _u32, C.POINTER(_vp)]),
    "cieg_matrix_upload_cuts": (_i, [_vp, C.POINTER(CsbView), _pu32, _u32, _u32, _pu32, _u32, C.POINTER(_vp)]),
    "cieg_pad_from_subspace": (_i, [_pd, _u32, _u32, _u32, _pd]),
    "cieg_multilevel_options_default": (None, [C.POINTER(MultilevelOptionsC)]),
    "cieg_multilevel_guess": (_i, [_vp, _vp, _pu32, _u32, C.POINTER(MultilevelOptionsC), _pd, _pu32,
                                   C.POINTER(LevelReportC)]),
    "cieg_lanczos_checkpoint": (_i, [C.c_int]),
    "cieg_lanczos_default_start": (_i, [_u32, _u32, _pd]),
    "cieg_lanczos_solve": (_i, [_vp, _vp, _pd, C.POINTER(LanczosOptionsC), C.POINTER(_vp)]),
    "cieg_lobpcg_solve_dist": (_i, [_vp, _vp, _pd, _u32, _vp, C.POINTER(LobpcgOptionsC), C.POINTER(DistHooks),
                                    C.POINTER(_vp)]),
    "cieg_lobpcg_solve_nccl": (_i, [_vp, _vp, _pd, _u32, _vp, C.POINTER(LobpcgOptionsC), C.POINTER(_vp)]),
    "cieg_nccl_unique_id": (_i, [C.POINTER(C.c_uint8)]),
    "cieg_ctx_nccl_init": (_i, [_vp, C.POINTER(C.c_uint8), _i, _i]),
    "cieg_ctx_nccl_finalize": (_i, [_vp]),
    "cieg_shard_plan": (_i, [C.POINTER(CsbView), _pu32, _u32, _u32, _u32, _pu32, _pu32, _pu32]),
    "cieg_matrix_upload_shard": (_i, [_vp, C.POINTER(CsbView), _pu32, _u32, _u32, _u32, _u32, C.POINTER(_vp)]),
    "cieg_matrix_rows": (_i, [_vp, _pu32, _pu32, _pu32, _pu32]),
    "cieg_precond_from_csb_range": (_i, [_vp, C.POINTER(CsbView), _pu32, _u32, _u32, _u32, C.POINTER(_vp)]),
    "cieg_ctx_set_stream": (_i, [_vp, _vp]),
    "cieg_ctx_set_exact_order": (_i, [_vp, _i]),
    "cieg_ctx_set_spmm_mode": (_i, [_vp, _i]),
    "cieg_spmm_effective_mode": (_i, [_vp, _vp, _u32, C.POINTER(C.c_int)]),
    "cieg_spmm_partial": (_i, [_vp, _vp, _vp, _vp, _u32, _vp]),
    "cieg_matrix_partial_rows": (_i, [_vp, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
    "cieg_report_summary": (_i, [_vp, _pi, _pi, _pd, _pu32, _pu32, _pu64]),
    "cieg_report_counters": (_i, [_vp, _pu64]),
    "cieg_report_eigenvalues": (_i, [_vp, _pd]),
    "cieg_report_trial_vectors": (_i, [_vp, _pd]),
    "cieg_report_history": (_i, [_vp, _pi, _pi, _pd, _pd]),
    "cieg_report_timing": (_i, [_vp, _pd]),
    "cieg_gen_expected_nnz": (_d, [C.POINTER(GenParams)]),
    "cieg_gen_avg_row_nnz": (_d, [C.POINTER(GenParams)]),
    "cieg_gen_count_nnz": (C.c_uint64, [C.POINTER(GenParams)]),
    "cieg_generate_csb": (_i, [C.POINTER(GenParams), C.POINTER(_vp)]),
    "cieg_host_csb_destroy": (_i, [_vp]),
    "cieg_host_csb_view": (_i, [_vp, C.POINTER(CsbView), _pu64]),
    "cieg_host_csb_groups": (_i, [_vp, C.POINTER(_pu32), _pu32]),
    "cieg_random_block": (_i, [_u32, _u32, _u64, _pd]),
    "cieg_generate_device": (_i, [_vp, C.POINTER(GenParams), _u32, _u32, _u32, C.POINTER(_vp)]),
    "cieg_generated_panels": (_i, [C.POINTER(GenParams), _u32, C.POINTER(_u32), _u32, C.POINTER(_u32)]),
    "cieg_precond_from_matrix": (_i, [_vp, _vp, C.POINTER(_vp)]),
    "cieg_matrix_groups": (_i, [_vp, C.POINTER(_pu32), _pu32]),
    "cieg_matrix_export": (_i, [_vp, _pu64, _pu32, _pu32, _pu32, _vp]),
}

_LIB = None


def load() -> C.CDLL:
    """Load libcieg.so (raises ImportError when it is missing -- no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the CUDA path has no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_LOCAL)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _LIB = lib
    return lib


def exported_symbols() -> list[str]:
    return list(SIGNATURES)
