"""ctypes bindings of the dlx C ABI (include/dlx.h) — the in-tree ``libdlx.so``.

There is no fallback: if the CUDA library is missing, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# DLX_LIB_PATH: an alternative build of the same library (A/B experiments of compile-time variants)
LIB_PATH = os.environ.get("DLX_LIB_PATH") or os.path.join(_HERE, "libdlx.so")

DLX_OK = 0
DLX_ERR_CUDA = 1
DLX_ERR_GENERATION = 2
DLX_ERR_TRAP = 3
DLX_ERR_ARG = 4
DLX_ERR_COMM = 5

KMEANS_AUTO, KMEANS_DIRECT, KMEANS_SCREENED = 0, 1, 2


class DlxError(RuntimeError):
    """Base class: a dlx entry point returned a non-zero status."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[dlx {code}] {msg}")
        self.code = code


class GenerationFailed(DlxError):
    """Mirrors stagekit StagingError::GenerationFailed (errors.hpp:19; codegen.cpp:66-71):
    the executor has no lowering for this loop / shape.  There is no CPU fallback."""


class TrapError(DlxError):
    """Mirrors stagekit TrapError (errors.hpp:46-67)."""


_lib = None

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_u64 = ctypes.c_uint64
_sz = ctypes.c_size_t
_int = ctypes.c_int
_dbl = ctypes.c_double

_SIGS = {
    "dlx_last_error": (ctypes.c_char_p, []),
    "dlx_version": (ctypes.c_char_p, []),
    "dlx_launch_count": (_u64, []),
    "dlx_device_count": (_int, [ctypes.POINTER(_int)]),
    "dlx_set_device": (_int, [_int]),
    "dlx_sm_count": (_int, [ctypes.POINTER(_int)]),
    "dlx_malloc": (_int, [ctypes.POINTER(_vp), _sz]),
    "dlx_free": (_int, [_vp]),
    "dlx_host_alloc": (_int, [ctypes.POINTER(_vp), _sz]),
    "dlx_host_free": (_int, [_vp]),
    "dlx_memcpy_h2d": (_int, [_vp, _vp, _sz, _vp]),
    "dlx_memcpy_d2h": (_int, [_vp, _vp, _sz, _vp]),
    "dlx_memset": (_int, [_vp, _int, _sz, _vp]),
    "dlx_stream_create": (_int, [ctypes.POINTER(_vp)]),
    "dlx_stream_destroy": (_int, [_vp]),
    "dlx_stream_sync": (_int, [_vp]),
    "dlx_rng_units": (_int, [_vp, _i64, _u64, _u64, _vp]),
    "dlx_rng_ints": (_int, [_vp, _i64, _i64, _u64, _u64, _vp]),
    "dlx_kmeans_workspace_bytes": (_sz, [_i64, _i32, _i32]),
    "dlx_kmeans_step": (_int, [_vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _sz, _int, _vp]),
    "dlx_kmeans_update": (_int, [_vp, _vp, _i32, _i32, _vp, _vp]),
    "dlx_kmeans_iteration": (_int, [_vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _sz, _int, _vp]),
    "dlx_kmeans_last_recheck_count": (_int, [_vp, _i64, _i32, _i32, ctypes.POINTER(_i64), _vp]),
    "dlx_groupby_workspace_bytes": (_sz, [_i64, _i64]),
    "dlx_groupby_count": (_int, [_vp, _i64, _i64, _vp, _vp, _sz, _vp]),
    "dlx_logreg_workspace_bytes": (_sz, [_i64, _i32]),
    "dlx_logreg_grad": (_int, [_vp, _vp, _i64, _i32, _vp, _vp, _vp, _sz, _vp]),
    "dlx_logreg_grad_f32": (_int, [_vp, _vp, _i64, _i32, _vp, _vp, _vp, _sz, _vp]),
    "dlx_axpy_inplace": (_int, [_vp, _vp, _dbl, _i64, _vp]),
    "dlx_rowdot_link_grad": (_int, [_vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "dlx_link_kind": (_int, [_vp]),
    "dlx_gda_workspace_bytes": (_sz, [_i64, _i32]),
    "dlx_gda_pass1": (_int, [_vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "dlx_gda_means": (_int, [_vp, _vp, _vp, _i64, _i32, _vp, _vp, _vp]),
    "dlx_gda_pass2": (_int, [_vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "dlx_map_axpy": (_int, [_dbl, _vp, _vp, _i64, _vp, _vp]),
    "dlx_reduce_workspace_bytes": (_sz, [_i64]),
    "dlx_reduce_sum_f64": (_int, [_vp, _i64, _vp, _vp, _sz, _vp]),
    "dlx_reduce_sum_i64": (_int, [_vp, _i64, _vp, _vp, _sz, _vp]),
    "dlx_reduce_sum_sumsq_f64": (_int, [_vp, _i64, _vp, _vp, _sz, _vp]),
    "dlx_reduce_count_gt_f64": (_int, [_vp, _i64, _dbl, _vp, _vp, _sz, _vp]),
    "dlx_widen_i32_i64": (_int, [_vp, _i64, _vp, _vp]),
    "dlx_vm_workspace_bytes": (_sz, [_i64]),
    "dlx_vm_run_loop": (_int, [_vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "dlx_bucket_rowsum_workspace_bytes": (_sz, [_i64, _i32, _i32]),
    "dlx_bucket_rowsum": (_int, [_vp, _vp, _i64, _i32, _vp, _i32, _vp, _vp, _vp, _sz, _vp]),
    "dlx_program_run": (_int, [ctypes.c_char_p, _u64, _int, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p)]),
    "dlx_program_create": (_int, [ctypes.c_char_p, _sz, ctypes.POINTER(_vp)]),
    "dlx_program_destroy": (_int, [_vp]),
    "dlx_program_execute": (_int, [_vp, _vp, _vp]),
    "dlx_run_result_free": (None, [_vp]),
    "dlx_string_free": (None, [_vp]),
    "dlx_comm_unique_id": (_int, [ctypes.c_char_p]),
    "dlx_comm_init": (_int, [ctypes.POINTER(_vp), ctypes.c_char_p, _int, _int]),
    "dlx_comm_destroy": (_int, [_vp]),
    "dlx_comm_allreduce_sum": (_int, [_vp, _vp, _i64, _int, _vp]),
    "dlx_comm_allreduce_sum_group": (_int, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_i64),
                                            ctypes.POINTER(_int), _int, _vp]),
    "dlx_gda_fit_workspace_bytes": (_sz, [_i64, _int]),
    "dlx_gda_fit": (_int, [_vp, _vp, _i64, _int, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "dlx_gda_combine_ranks": (_int, [_vp, _int, _int, _vp, _vp, _vp, _vp, _vp]),
    "dlx_gda_fit_last_fallback": (_int, [_vp, _i64, _int, ctypes.POINTER(_int)]),
    "dlx_gda_fit_path": (_int, [_vp, _vp, _i64, _int, ctypes.POINTER(_int)]),
    "dlx_peer_alloc": (_int, [_i64, ctypes.POINTER(_vp), ctypes.c_char_p]),
    "dlx_peer_open": (_int, [ctypes.c_char_p, ctypes.POINTER(_vp)]),
    "dlx_peer_close": (_int, [_vp]),
    "dlx_peer_free": (_int, [_vp]),
    "dlx_peer_allreduce": (_int, [ctypes.POINTER(_vp), _int, _int, _i64, _i64, _int, _int, _vp, _vp,
                                  _int, _vp, _dbl, _vp]),
}

# Every symbol include/dlx*.h declares (checked by tests/test_abi.py).
EXPORTED = tuple(_SIGS)


def load():
    """Load libdlx.so and set the argument types.  Raises if the library is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    for name, (res, args) in _SIGS.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(rc: int) -> None:
    if rc == DLX_OK:
        return
    msg = load().dlx_last_error().decode(errors="replace")
    if rc == DLX_ERR_GENERATION:
        raise GenerationFailed(rc, msg)
    if rc == DLX_ERR_TRAP:
        raise TrapError(rc, msg)
    raise DlxError(rc, msg)


# ---- dlx_program.h structs --------------------------------------------------------------------
VAL_UNIT, VAL_INT, VAL_DOUBLE, VAL_BOOL, VAL_STR, VAL_VECTOR = range(6)
EXEC_SERIAL, EXEC_DRYRUN, EXEC_NOCACHE = 1, 2, 4


class ProgramInput(ctypes.Structure):
    _fields_ = [("sym", _i32), ("elem", _i32), ("n", _i64), ("h_data", _vp), ("d_data", _vp)]


class ExecOptions(ctypes.Structure):
    _fields_ = [("seed", _u64), ("ndevices", _i32), ("devices", ctypes.POINTER(_i32)), ("ninputs", _i32),
                ("inputs", ctypes.POINTER(ProgramInput)), ("flags", _i32)]


class RunResult(ctypes.Structure):
    _fields_ = [("text", _vp), ("report", _vp), ("kind", _i32), ("i", _i64), ("d", _dbl), ("s", _vp),
                ("vec_elem", _i32), ("vec_len", _i64), ("vec_data", _vp)]
