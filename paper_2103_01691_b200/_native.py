"""ctypes binding of ``libkmb200.so`` (the C ABI declared in include/kmb200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``make -C
paper_2103_01691_b200/csrc``).  There is no CPU fallback: every public entry
point that computes goes through :func:`lib`, which raises
:class:`NativeLibraryError` when the shared object is missing.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ConfigurationError, DeviceError, NativeLibraryError

# KMB200_LIB overrides the library path (A/B builds of the same ABI)
LIB_PATH = os.environ.get("KMB200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libkmb200.so")
ABI_VERSION = 3
MAX_D = 8

KM_F32, KM_F64, KM_C64, KM_C128 = 0, 1, 2, 3
KM_OK, KM_EINVAL, KM_ECUDA = 0, 1, 2
OP_NONE, OP_GPE_PHASE, OP_DIAG = 0, 1, 2
POLICY_AUTO, POLICY_NO_TMA, POLICY_NO_STREAMK, POLICY_NO_TC_HALVES, POLICY_NO_PLANE_FUSION = 0, 1, 2, 4, 8

# every symbol include/kmb200.h declares
EXPORTS = (
    "km_abi_version",
    "km_build_info",
    "km_last_error",
    "km_mumode",
    "km_mumode_split",
    "km_mumode_fibers",
    "km_copy_2d",
    "km_diag_phase_fold",
    "km_mumode_peer",
    "km_tucker",
    "km_tucker_workspace",
    "km_pointwise",
    "km_pointwise_cast",
    "km_set_kernel_policy",
    "km_tc_workspace_bytes",
    "km_mumode_c64_tc",
    "km_norm_workspace_bytes",
    "km_norm",
    "km_stream_workspace_bytes",
    "km_steps_small_workspace_bytes",
    "km_steps_small",
    "km_steps_paired",
    "km_norm_epilogue_slots",
    "km_set_stream_workspace",
)


class PointOp(ctypes.Structure):
    """Mirror of ``km_pointop`` (include/kmb200.h)."""

    _fields_ = [
        ("kind", ctypes.c_int32),
        ("d", ctypes.c_int32),
        ("dims", ctypes.c_int64 * MAX_D),
        ("weights", ctypes.c_void_p * MAX_D),
        ("coef", ctypes.c_double),
        ("diag", ctypes.c_void_p),
        ("diag_dir", ctypes.c_int32),
        ("repeat", ctypes.c_int32),
        ("inner_weights", ctypes.c_void_p),
        ("norm_result", ctypes.c_void_p),
        ("norm_ws", ctypes.c_void_p),
        ("norm_ws_count", ctypes.c_int64),
    ]


_lock = threading.Lock()
_lib = None


def _declare(lib):
    c_int, c_i64, c_vp, c_sz = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t
    p_op = ctypes.POINTER(PointOp)
    lib.km_abi_version.restype = c_int
    lib.km_abi_version.argtypes = []
    lib.km_build_info.restype = ctypes.c_char_p
    lib.km_build_info.argtypes = []
    lib.km_last_error.restype = ctypes.c_char_p
    lib.km_last_error.argtypes = []
    lib.km_mumode.restype = c_int
    lib.km_mumode.argtypes = [c_vp, c_int, c_vp, c_int, c_vp, c_i64, c_i64, c_i64, c_i64, p_op, c_vp]
    lib.km_mumode_split.restype = c_int
    lib.km_mumode_split.argtypes = [c_vp, c_int, c_vp, c_int, c_vp, c_i64, c_i64, c_i64, c_i64,
                                    ctypes.c_int32, c_i64, ctypes.c_int32, c_i64, ctypes.c_int32, p_op, c_vp]
    lib.km_mumode_fibers.restype = c_int
    lib.km_mumode_fibers.argtypes = [c_vp, c_int, c_vp, c_int, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp]
    lib.km_diag_phase_fold.restype = c_int
    lib.km_diag_phase_fold.argtypes = [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, ctypes.c_double, ctypes.c_double, c_vp]
    lib.km_copy_2d.restype = c_int
    lib.km_copy_2d.argtypes = [c_vp, c_sz, c_vp, c_sz, c_sz, c_sz, c_vp]
    lib.km_mumode_peer.restype = c_int
    lib.km_mumode_peer.argtypes = [c_vp, c_int, c_vp, c_int, c_i64, c_i64, c_i64, c_i64, ctypes.c_int32, c_i64,
                                   ctypes.c_int32, c_i64, ctypes.POINTER(c_vp), ctypes.c_int32, c_i64, c_vp]
    lib.km_tucker.restype = c_int
    lib.km_tucker.argtypes = [
        c_vp, c_int, c_int, ctypes.POINTER(c_i64), ctypes.POINTER(c_vp), ctypes.POINTER(c_int),
        ctypes.POINTER(c_i64), c_vp, c_vp, c_vp, p_op, p_op, c_vp,
    ]
    lib.km_tucker_workspace.restype = c_int
    lib.km_tucker_workspace.argtypes = [
        c_int, c_int, ctypes.POINTER(c_i64), ctypes.POINTER(c_vp), ctypes.POINTER(c_int),
        ctypes.POINTER(c_i64), ctypes.POINTER(c_sz),
    ]
    lib.km_tc_workspace_bytes.restype = c_int
    lib.km_tc_workspace_bytes.argtypes = [c_i64, c_i64, ctypes.POINTER(c_sz)]
    lib.km_mumode_c64_tc.restype = c_int
    lib.km_mumode_c64_tc.argtypes = [c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_sz, c_vp]
    lib.km_norm_workspace_bytes.restype = c_sz
    lib.km_norm_workspace_bytes.argtypes = []
    lib.km_norm.restype = c_int
    lib.km_norm.argtypes = [c_vp, c_vp, c_int, c_i64, c_int, p_op, c_vp, c_vp, c_sz, c_vp]
    lib.km_set_kernel_policy.restype = c_int
    lib.km_set_kernel_policy.argtypes = [c_int]
    lib.km_steps_small_workspace_bytes.restype = c_int
    lib.km_steps_small_workspace_bytes.argtypes = [c_i64, c_i64, c_i64, c_i64, ctypes.POINTER(c_sz)]
    lib.km_norm_epilogue_slots.restype = c_i64
    lib.km_norm_epilogue_slots.argtypes = [c_i64, c_i64]
    lib.km_steps_small.restype = c_int
    lib.km_steps_small.argtypes = [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_sz, c_vp]
    lib.km_steps_paired.restype = c_int
    lib.km_steps_paired.argtypes = [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]
    lib.km_stream_workspace_bytes.restype = c_int
    lib.km_stream_workspace_bytes.argtypes = [ctypes.POINTER(c_sz)]
    lib.km_set_stream_workspace.restype = c_int
    lib.km_set_stream_workspace.argtypes = [c_vp, c_vp, c_sz]
    lib.km_pointwise.restype = c_int
    lib.km_pointwise.argtypes = [c_vp, c_vp, c_int, c_i64, p_op, c_vp]
    lib.km_pointwise_cast.restype = c_int
    lib.km_pointwise_cast.argtypes = [c_vp, c_int, c_vp, c_int, c_i64, p_op, c_vp]


PLANE_EXTENTS = (32, 48, 64)


def plane_fused(u_code, dims, mat_codes, rows):
    """Whether km_tucker runs the first two products of this step as one fused launch
    (csrc/kmb200_plane.cuh: d = 3 complex128, square complex128 E1/E2, planes of 32/48/64 on
    each side) under the default kernel policy; launch counts use it."""
    return (len(dims) == 3 and u_code == KM_C128 and len(mat_codes) == 3 and all(r > 0 for r in rows)
            and mat_codes[0] == KM_C128 and mat_codes[1] == KM_C128
            and rows[0] == dims[0] and rows[1] == dims[1]
            and dims[0] in PLANE_EXTENTS and dims[1] in PLANE_EXTENTS and dims[2] >= 1)


def lib():
    """The loaded library (loads on first use; raises if it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryError(
                    f"{LIB_PATH} is missing; build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)"
                )
            try:
                handle = ctypes.CDLL(LIB_PATH)
            except OSError as exc:
                raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
            missing = [s for s in EXPORTS if not hasattr(handle, s)]
            if missing:
                raise NativeLibraryError(f"{LIB_PATH} lacks symbols {missing}; rebuild it")
            _declare(handle)
            if handle.km_abi_version() != ABI_VERSION:
                raise NativeLibraryError(
                    f"{LIB_PATH} has ABI {handle.km_abi_version()}, expected {ABI_VERSION}; rebuild it"
                )
            _lib = handle
    return _lib


def check(rc):
    """Map a C status code to the exception hierarchy."""
    if rc == KM_OK:
        return
    msg = (lib().km_last_error() or b"").decode(errors="replace")
    if rc == KM_EINVAL:
        raise ConfigurationError(msg)
    raise DeviceError(msg)
