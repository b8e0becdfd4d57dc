"""ctypes binding of libpolynewt_b200.so (include/polynewt_b200.h).

The library is built in-tree (paper_1402_2626_b200/lib/) by
``__graft_entry__.build()`` / ``make -C paper_1402_2626_b200/csrc``.  There is
no CPU fallback: if the library or a CUDA device is missing, the calls that
need them raise.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PN_LIB selects an alternative build (performance experiments only)
LIB_PATH = os.environ.get("PN_LIB") or os.path.join(_HERE, "lib", "libpolynewt_b200.so")

PN_OK = 0
PN_E_ARG = 1
PN_E_BREAKDOWN = 2
PN_E_SINGULAR = 3
PN_E_DOMAIN = 4
PN_E_CUDA = 5
PN_E_NOMEM = 6
PN_E_COMM = 7

OP_ADD, OP_SUB, OP_MUL, OP_DIV, OP_ABS2, OP_SQRT, OP_CONJ, OP_MODULUS, OP_DIV_REAL = range(9)

_c_double_p = ctypes.POINTER(ctypes.c_double)
_c_int32_p = ctypes.POINTER(ctypes.c_int32)
_c_int64_p = ctypes.POINTER(ctypes.c_int64)


class NumInfo(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("index", ctypes.c_int32), ("rkk", ctypes.c_double),
                ("threshold", ctypes.c_double), ("z", ctypes.c_double), ("t_evaluate", ctypes.c_double),
                ("t_solve", ctypes.c_double), ("t_update", ctypes.c_double), ("t_factor", ctypes.c_double)]


class Counts(ctypes.Structure):
    _fields_ = [("eval_mults", ctypes.c_int64), ("grad_mults", ctypes.c_int64)]


class SystemStats(ctypes.Structure):
    _fields_ = [("nc", ctypes.c_int32), ("cplx", ctypes.c_int32), ("m", ctypes.c_int32), ("n", ctypes.c_int32),
                ("monomials", ctypes.c_int64), ("support", ctypes.c_int64), ("segments", ctypes.c_int64),
                ("mul_ops", ctypes.c_int64), ("int_mul_ops", ctypes.c_int64), ("add_ops", ctypes.c_int64),
                ("table_mul_ops", ctypes.c_int64), ("max_k", ctypes.c_int32), ("max_deg", ctypes.c_int32)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("rows_ok", ctypes.c_int32), ("K", ctypes.c_int32), ("chunk", ctypes.c_int32),
                ("depth", ctypes.c_int32), ("nchunks", ctypes.c_int64)]


# exported symbols and their signatures (argtypes, restype)
SIGNATURES = {
    "pn_version": ([], ctypes.c_int),
    "pn_last_error": ([], ctypes.c_char_p),
    "pn_device_count": ([ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "pn_launch_count": ([], ctypes.c_int64),
    "pn_fp64_peak": ([ctypes.POINTER(ctypes.c_double), ctypes.c_void_p], ctypes.c_int),
    "pn_vec_op": ([ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                   ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "pn_tree_sum": ([ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
                    ctypes.c_int),
    "pn_system_create": ([ctypes.c_int, ctypes.c_int, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64,
                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                          ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "pn_system_destroy": ([ctypes.c_void_p], ctypes.c_int),
    "pn_system_get_stats": ([ctypes.c_void_p, ctypes.POINTER(SystemStats)], ctypes.c_int),
    "pn_parse_system": ([ctypes.c_char_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)],
                        ctypes.c_int),
    "pn_text_system_sizes": ([ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                              ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
    "pn_text_system_export": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.c_void_p], ctypes.c_int),
    "pn_text_system_free": ([ctypes.c_void_p], ctypes.c_int),
    "pn_comm_unique_id": ([ctypes.c_void_p], ctypes.c_int),
    "pn_comm_init": ([ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)],
                     ctypes.c_int),
    "pn_comm_destroy": ([ctypes.c_void_p], ctypes.c_int),
    "pn_batch_allgather": ([ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int32, ctypes.c_int64,
                            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                            ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "pn_system_plan_info": ([ctypes.c_void_p, ctypes.POINTER(PlanInfo)], ctypes.c_int),
    "pn_system_canonical_order": ([ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "pn_system_counts": ([ctypes.c_void_p, ctypes.POINTER(Counts)], ctypes.c_int),
    "pn_evaldiff": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(Counts),
                     ctypes.c_void_p], ctypes.c_int),
    "pn_mgs_qr": ([ctypes.c_int, ctypes.c_int, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                   ctypes.c_void_p, ctypes.POINTER(NumInfo), ctypes.c_void_p], ctypes.c_int),
    "pn_back_substitute": ([ctypes.c_int, ctypes.c_int, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                            ctypes.POINTER(NumInfo), ctypes.c_void_p], ctypes.c_int),
    "pn_least_squares": ([ctypes.c_int, ctypes.c_int, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p,
                          ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p, ctypes.c_void_p,
                          ctypes.POINTER(NumInfo), ctypes.c_void_p], ctypes.c_int),
    "pn_residual_check": ([ctypes.c_int, ctypes.c_int, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p],
                          ctypes.c_int),
    "pn_newton_step": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(NumInfo), ctypes.c_void_p],
                       ctypes.c_int),
    "pn_newton_batch": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                         ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
                        ctypes.c_int),
    "pn_evaldiff_batch": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
                          ctypes.c_int),
    "pn_generate_random_system": ([ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                   ctypes.c_int32, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
}

_lib = None
_lock = threading.Lock()


class LibraryMissingError(ImportError):
    pass


def load():
    """Load the shared library (once); raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise LibraryMissingError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "or `make -C paper_1402_2626_b200/csrc` (no CPU fallback exists)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (argtypes, restype) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = argtypes
                fn.restype = restype
            _lib = lib
    return _lib


def last_error() -> str:
    msg = load().pn_last_error()
    return msg.decode() if msg else ""


def device_count() -> int:
    c = ctypes.c_int(0)
    load().pn_device_count(ctypes.byref(c))
    return c.value


def require_gpu():
    if device_count() < 1:
        raise RuntimeError("polynewt_b200 needs a CUDA device (no CPU fallback)")


def launch_count() -> int:
    return int(load().pn_launch_count())


def ptr(a) -> ctypes.c_void_p:
    """Data pointer of a C-contiguous float64/int array, a torch tensor, or None."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("arrays passed to the C ABI must be C-contiguous")
        return ctypes.c_void_p(a.ctypes.data)
    if hasattr(a, "data_ptr"):  # torch tensor (host or device)
        if not a.is_contiguous():
            raise ValueError("tensors passed to the C ABI must be contiguous")
        return ctypes.c_void_p(a.data_ptr())
    raise TypeError(f"cannot pass {type(a).__name__} to the C ABI")


def check(rc: int, info: NumInfo | None = None):
    """Map a status code onto the reference's exception types."""
    if rc == PN_OK:
        return
    msg = last_error()
    if rc == PN_E_ARG:
        raise ValueError(msg)
    if rc == PN_E_BREAKDOWN:
        from .mgs import MgsBreakdownError
        raise MgsBreakdownError(info.k, info.rkk, info.threshold)
    if rc == PN_E_SINGULAR:
        from .mgs import SingularMatrixError
        raise SingularMatrixError(info.index)
    if rc == PN_E_DOMAIN:
        from .xprec import DomainError
        raise DomainError(msg)
    if rc == PN_E_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg or f"polynewt_b200 error {rc}")
