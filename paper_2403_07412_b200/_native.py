"""ctypes binding of libvecchia_b200.so (C ABI in include/vecchia_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``make -C
paper_2403_07412_b200/csrc``).  There is deliberately no fallback: if the
shared object is missing this module raises at import, and every compute call
raises :class:`NativeError` when no CUDA device is usable.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import (
    LikelihoodEvaluationError,
    NonPositiveDefiniteError,
    SingularTriangularError,
    VecchiaGPError,
)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libvecchia_b200.so")

VGP_OK = 0
VGP_NOT_POSITIVE_DEFINITE = 1
VGP_BAD_CONDITIONAL_VARIANCE = 2
VGP_SINGULAR_TRIANGULAR = 3
VGP_E_INVALID = -1
VGP_E_CUDA = -2
VGP_E_NOMEM = -3
VGP_E_UNSUPPORTED = -4

FAMILY_CODES = {"matern": 0, "power_exponential": 1}
METRIC_EUCLIDEAN = 0
METRIC_GREAT_CIRCLE = 1

# Every symbol include/vecchia_b200.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "vgp_version", "vgp_last_error", "vgp_device_count", "vgp_knn_predecessors",
    "vgp_knn_points", "vgp_cov", "vgp_bessel_kv", "vgp_plan_create", "vgp_plan_set_data",
    "vgp_plan_destroy", "vgp_loglik", "vgp_loglik_partials", "vgp_plan_info",
    "vgp_plan_set_variant", "vgp_plan_stream", "vgp_loglik_async", "vgp_plan_fetch",
    "vgp_host_register", "vgp_host_unregister", "vgp_krige", "vgp_knn_sphere",
    "vgp_batch_potrf", "vgp_batch_trsv", "vgp_batch_dot", "vgp_loglik_partials_device",
    "vgp_plan_set_timing", "vgp_plan_kernel_time", "vgp_maxmin_order", "vgp_assemble",
    "vgp_simulate", "vgp_knn_predecessors_range",
    "vgp_plan_create_shard", "vgp_plan_fail_keys", "vgp_loglik_data",
)


class NativeError(VecchiaGPError, RuntimeError):
    """A CUDA / argument failure inside libvecchia_b200 (negative status)."""

    def __init__(self, code: int, msg: str):
        self.code = code
        super().__init__(f"libvecchia_b200 error {code}: {msg}")


if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "or `make -C paper_2403_07412_b200/csrc`; the B200 path has no CPU fallback"
    )

lib = ctypes.CDLL(LIB_PATH)

_d = ctypes.c_double
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_int = ctypes.c_int
_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int64)
_vp = ctypes.c_void_p


def _sig(name, restype, argtypes):
    f = getattr(lib, name)
    f.restype = restype
    f.argtypes = argtypes
    return f


_sig("vgp_version", ctypes.c_char_p, [])
_sig("vgp_last_error", ctypes.c_char_p, [])
_sig("vgp_device_count", _int, [ctypes.POINTER(_int)])
_sig("vgp_knn_predecessors", _int, [_int, _dp, _i64, _i32, _ip])
_sig("vgp_knn_points", _int, [_int, _dp, _i64, _dp, _i64, _i32, _ip])
_sig("vgp_cov", _int, [_int, _int, _d, _d, _d, _dp, _i64, _dp])
_sig("vgp_bessel_kv", _int, [_int, _d, _dp, _i64, _dp])
_sig("vgp_plan_create", _int, [_int, _i64, _i32, _int, _d, _ip, _ip, _i64, _i64,
                               ctypes.POINTER(_vp)])
_sig("vgp_plan_set_data", _int, [_vp, _dp, _dp])
_sig("vgp_host_register", _int, [_vp, _i64])
_sig("vgp_knn_sphere", _int, [_int, _dp, _i64, _dp, _i64, _i32, _int, _ip])
_sig("vgp_krige", _int, [_int, _dp, _dp, _i64, _dp, _i64, _i32, _ip, _int, _d, _int, _d, _d, _d,
                         _dp, _dp, _ip])
_sig("vgp_host_unregister", _int, [_vp])
_sig("vgp_maxmin_order", _int, [_int, _dp, _i64, _i64, _ip])
_sig("vgp_assemble", _int, [_int, _dp, _dp, _i64, _i32, _ip, _int, _d, _int, _d, _d, _d, _dp, _i64, _dp,
                            _i64, _dp, _i64])
_sig("vgp_plan_destroy", _int, [_vp])
_sig("vgp_loglik", _int, [_vp, _int, _d, _d, _d, _dp, _ip, _dp, _dp, _dp, _dp])
_sig("vgp_knn_predecessors_range", _int, [_int, _dp, _i64, _i32, _i64, _i64, _ip])
_sig("vgp_plan_create_shard", _int, [_int, _i64, _i32, _int, _d, _ip, _ip, _i64, _i64,
                                    ctypes.POINTER(_vp)])
_sig("vgp_plan_fail_keys", _int, [_vp, ctypes.POINTER(ctypes.c_uint64)])
_sig("vgp_loglik_data", _int, [_vp, _dp, _dp, _int, _d, _d, _d, _dp, _ip, _dp, _dp, _dp, _dp])
_sig("vgp_simulate", _int, [_vp, _int, _d, _d, _d, _dp, _dp, _ip])
_sig("vgp_loglik_partials", _int, [_vp, _int, _d, _d, _d, _dp, _dp, _ip])
_sig("vgp_plan_info", _int, [_vp, _ip])
_sig("vgp_plan_set_variant", _int, [_vp, _int])
_sig("vgp_plan_stream", _vp, [_vp])
_sig("vgp_loglik_async", _int, [_vp, _int, _d, _d, _d])
_sig("vgp_plan_fetch", _int, [_vp, _dp, _ip, ctypes.POINTER(_int)])
_sig("vgp_loglik_partials_device", _int, [_vp, _int, _d, _d, _d, _vp])
_sig("vgp_plan_set_timing", _int, [_vp, _int])
_sig("vgp_plan_kernel_time", _int, [_vp, _dp, _ip])
_sig("vgp_batch_potrf", _int, [_int, _dp, _i64, _i32, _i64, _ip])
_sig("vgp_batch_trsv", _int, [_int, _dp, _i64, _dp, _dp, _i64, _i32, _i64, _ip])
_sig("vgp_batch_dot", _int, [_int, _dp, _dp, _i64, _i32, _i64, _dp])


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def iptr(a: np.ndarray):
    return a.ctypes.data_as(_ip)


def null_d():
    return ctypes.cast(None, _dp)


def last_error() -> str:
    return lib.vgp_last_error().decode(errors="replace")


def check(rc: int) -> int:
    """Raise NativeError for negative status codes; pass through the rest."""
    if rc < 0:
        raise NativeError(rc, last_error())
    return rc


def raise_for_status(rc: int, fail_index: int, where: str = "") -> None:
    """Map positive statuses to the reference's exception types."""
    if rc == VGP_OK:
        return
    if rc == VGP_NOT_POSITIVE_DEFINITE:
        # _numeric_stage re-raises NPD as LikelihoodEvaluationError (vg/vecchia.py:182-185)
        exc = NonPositiveDefiniteError(fail_index, where)
        raise LikelihoodEvaluationError(fail_index, str(exc)) from exc
    if rc == VGP_BAD_CONDITIONAL_VARIANCE:
        raise LikelihoodEvaluationError(fail_index, f"conditional variance <= 0 {where}".strip())
    if rc == VGP_SINGULAR_TRIANGULAR:
        raise SingularTriangularError(fail_index)
    check(rc)


def device_count() -> int:
    c = _int(0)
    lib.vgp_device_count(ctypes.byref(c))
    return int(c.value)


def version() -> str:
    return lib.vgp_version().decode()


_device = [None]


def current_device() -> int:
    """CUDA ordinal this process drives (LOCAL_RANK under torchrun, else 0)."""
    if _device[0] is None:
        _device[0] = int(os.environ.get("VGP_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    return _device[0]


def set_device(dev: int) -> None:
    _device[0] = int(dev)
