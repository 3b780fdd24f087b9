"""ctypes binding of the C ABI in include/pfe_b200.h (libpfe_b200.so).

The library is the product: every compute entry point runs sm_100a kernels.
There is no Python or CPU fallback — if the shared library is missing or no
sm_100-class GPU is present, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libpfe_b200.so"
# A/B experiments only: PFE_LIB_VARIANT=<name> loads lib_<name>/libpfe_b200.so
# (an in-tree build of a modified source tree, scripts/build_variant.sh)
if os.environ.get("PFE_LIB_VARIANT"):
    LIB_PATH = Path(__file__).resolve().parent / f"lib_{os.environ['PFE_LIB_VARIANT']}" / "libpfe_b200.so"

PFE_OK, PFE_IO_ERROR, PFE_NUMERICAL_ERROR, PFE_CONFIG_ERROR, PFE_CUDA_ERROR = 0, 1, 2, 3, 4


class pfe_graph(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int64), ("ei", C.POINTER(C.c_int32)), ("ej", C.POINTER(C.c_int32)),
                ("w", C.POINTER(C.c_double)), ("degree", C.POINTER(C.c_double)), ("grid_h", C.c_int32),
                ("grid_w", C.c_int32), ("grid_radius", C.c_int32)]


class pfe_params(C.Structure):
    _fields_ = [("dim", C.c_int32), ("lambda_", C.c_double), ("r", C.c_double), ("soc_max", C.c_int32),
                ("sb_max_stage1", C.c_int32), ("sb_max_stage2", C.c_int32), ("conv_tol", C.c_double),
                ("pcg_rel_tol", C.c_double), ("pcg_max_iter", C.c_int32), ("preconditioner", C.c_int32)]


class pfe_exec(C.Structure):
    _fields_ = [("device", C.c_int32), ("use_graphs", C.c_int32), ("warn", C.c_int32), ("profile", C.c_int32),
                ("persistent", C.c_int32)]


class pfe_report(C.Structure):
    _fields_ = [("inner_iterations", C.c_int64), ("pcg_iterations", C.c_int64),
                ("pcg_column_iterations", C.c_int64), ("nonconverged", C.c_int64), ("failed", C.c_int64),
                ("jacobi_fallback", C.c_int32), ("topology", C.c_int32), ("n", C.c_int64), ("m", C.c_int64),
                ("d", C.c_int32), ("persistent_kind", C.c_int32), ("setup_seconds", C.c_double)]


KERNEL_CLASSES = ("pcg_init", "pcg_spmv", "pcg_update", "pcg_finalize", "sb_pass", "rhs", "projection",
                  "sb_persistent")


class pfe_kernel_times(C.Structure):
    _fields_ = [("ms", C.c_double * 8), ("launches", C.c_int64 * 8)]


ITERATE_FN = C.CFUNCTYPE(None, C.c_int, C.POINTER(C.c_double), C.c_int32, C.c_int32, C.c_void_p)

_P = C.c_void_p
_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int32)

_SIGS = {
    "pfe_last_error": (C.c_char_p, []),
    "pfe_release_cached_memory": (C.c_int64, [C.c_int32]),
    "pfe_params_default": (pfe_params, []),
    "pfe_exec_default": (pfe_exec, []),
    "pfe_device_check": (C.c_int, [C.c_int32]),
    "pfe_solver_create": (C.c_int, [C.POINTER(pfe_graph), C.POINTER(pfe_params), C.POINTER(pfe_exec),
                                    C.POINTER(_P)]),
    "pfe_solver_destroy": (None, [_P]),
    "pfe_solver_report": (C.c_int, [_P, C.POINTER(pfe_report)]),
    "pfe_solver_pcg_log": (C.c_int64, [_P, _I, _I, _D, C.c_int64]),
    "pfe_solver_kernel_times": (C.c_int, [_P, C.POINTER(pfe_kernel_times), C.c_int]),
    "pfe_solver_last_ms": (C.c_double, [_P]),
    "pfe_solver_trace": (C.c_int64, [_P, C.POINTER(C.c_uint64), C.c_int64]),
    "pfe_state_create": (C.c_int, [_P, _D, C.POINTER(_P)]),
    "pfe_state_reset": (C.c_int, [_P]),
    "pfe_state_destroy": (None, [_P]),
    "pfe_state_get": (C.c_int, [_P, C.c_int32, _D]),
    "pfe_state_set": (C.c_int, [_P, C.c_int32, _D]),
    "pfe_split_bregman": (C.c_int, [_P, _P, C.c_int32, ITERATE_FN, C.c_void_p]),
    "pfe_run_soc": (C.c_int, [_P, _P, C.c_int32, C.c_int32]),
    "pfe_two_stage": (C.c_int, [_P, _P]),
    "pfe_state_objective": (C.c_int, [_P, _P, _D]),
    "pfe_solve": (C.c_int, [C.POINTER(pfe_graph), C.POINTER(pfe_params), C.POINTER(pfe_exec), C.c_int32, _D, _D,
                            C.POINTER(pfe_report)]),
    "pfe_split_bregman_standalone": (C.c_int, [C.POINTER(pfe_graph), _D, _D, C.POINTER(pfe_params), C.c_int32, _D,
                                               C.c_int32, C.POINTER(pfe_exec), _D, ITERATE_FN, C.c_void_p]),
    "pfe_pcg_solve_multi": (C.c_int, [C.c_int32, _I, _I, _D, C.c_int32, _D, _D, C.c_double, C.c_int32, C.c_int32,
                                      C.POINTER(pfe_exec), _D, _I, _I, _D, _I]),
    "pfe_range_partition_stats": (C.c_int, [C.POINTER(pfe_graph), C.c_int32, C.POINTER(C.c_int64),
                                            C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "pfe_ic0_probe": (C.c_int, [C.c_int32, _I, _I, _D, _I]),
    "pfe_objective": (C.c_int, [C.POINTER(pfe_graph), C.c_int32, _D, C.POINTER(pfe_exec), _D]),
    "pfe_shrink": (C.c_int, [C.c_int64, _D, C.c_double, C.POINTER(pfe_exec), _D]),
    "pfe_project_orthogonal": (C.c_int, [C.c_int32, C.c_int32, _D, C.POINTER(pfe_exec), _D]),
    "pfe_band_plan": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, _I]),
    "pfe_nccl_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "pfe_solver_create_band": (C.c_int, [C.POINTER(pfe_graph), C.POINTER(pfe_params), C.POINTER(pfe_exec),
                                         C.POINTER(C.c_uint8), C.c_int32, C.c_int32, C.POINTER(_P)]),
    "pfe_solve_banded": (C.c_int, [C.POINTER(pfe_graph), C.POINTER(pfe_params), C.POINTER(pfe_exec), C.c_int32,
                                   C.c_int32, _D, _D, C.POINTER(pfe_report)]),
    "pfe_solve_multi_gpu": (C.c_int, [C.POINTER(pfe_graph), C.POINTER(pfe_params), C.POINTER(pfe_exec), C.c_int32,
                                      _I, C.c_int32, _D, _D, C.POINTER(pfe_report), _D]),
    "pfe_d_orthonormalize": (C.c_int, [C.c_int32, C.c_int32, _D, _D, _D]),
    "pfe_random_embedding": (C.c_int, [C.c_int32, C.c_int32, C.c_uint64, _D, _D]),
    "pfe_kmeans": (C.c_int, [C.c_int32, C.c_int32, _D, C.c_int32, C.c_uint64, C.c_int32, _I]),
    "pfe_kmeans_device": (C.c_int, [C.c_int32, C.c_int32, _D, C.c_int32, C.c_uint64, C.c_int32, C.c_int32, _I]),
    "pfe_gmm_init_device": (C.c_int, [C.c_int32, _D, C.c_int32, C.c_uint64, _D, C.c_int32, _D, _D, _D, _D]),
    "pfe_knn_graph": (C.c_int, [C.c_int32, C.c_int32, _D, C.c_int32, C.c_int32, _I, _I, _D, _D,
                                C.POINTER(C.c_int64), _D]),
    "pfe_grid_graph": (C.c_int, [C.c_int32, C.c_int32, _D, C.c_double, C.c_int32, C.c_double, C.c_int32, _I, _I,
                                 _D, _D, C.POINTER(C.c_int64)]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None


def load() -> C.CDLL:
    """Loads libpfe_b200.so (built by ``__graft_entry__.build()``); raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(f"{LIB_PATH} is missing: build the sm_100a library first "
                           "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_D)


def iptr(a: np.ndarray):
    return a.ctypes.data_as(_I)
