"""CPU: the C-ABI library loads, exports every symbol include/kmb200.h
declares, and rejects bad arguments before touching the device."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import HAS_CUDA, ROOT
from paper_2103_01691_b200 import _native

HEADER = os.path.join(ROOT, "include", "kmb200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|size_t|const char\*)\s+(km_\w+)\s*\(", text, re.M)))


def test_header_declares_the_binding_exports():
    assert declared_symbols() == sorted(_native.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    lib = _native.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.km_abi_version() == _native.ABI_VERSION
    assert b"sm_100a" in lib.km_build_info()


def test_library_is_sm100a_cubin():
    import subprocess

    out = subprocess.run(["cuobjdump", "-lelf", _native.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_struct_layout_matches_header():
    # km_pointop: 2*int32 + 8*int64 + 8*ptr + double + ptr + 2*int32 + ptr + 2*ptr + int64
    assert ctypes.sizeof(_native.PointOp) == 8 + 64 + 64 + 8 + 8 + 8 + 8 + 16 + 8


def test_bad_dtype_rejected_without_device():
    lib = _native.lib()
    rc = lib.km_mumode(None, 7, None, 3, None, 2, 1, 2, 1, None, None)
    assert rc == _native.KM_EINVAL
    assert b"dtype" in lib.km_last_error()


def test_mixed_precision_rejected():
    lib = _native.lib()
    dummy = ctypes.c_void_p(16)
    rc = lib.km_mumode(dummy, _native.KM_C64, dummy, _native.KM_C128, dummy, 2, 1, 2, 1, None, None)
    assert rc == _native.KM_EINVAL
    assert b"precision" in lib.km_last_error()


def test_nonpositive_extent_rejected():
    lib = _native.lib()
    dummy = ctypes.c_void_p(16)
    rc = lib.km_mumode(dummy, _native.KM_C128, dummy, _native.KM_C128, dummy, 0, 1, 2, 1, None, None)
    assert rc == _native.KM_EINVAL


def test_bad_op_rejected():
    lib = _native.lib()
    dummy = ctypes.c_void_p(16)
    op = _native.PointOp()
    op.kind = 9
    op.d = 3
    rc = lib.km_mumode(dummy, _native.KM_C128, dummy, _native.KM_C128, dummy, 2, 1, 2, 1,
                       ctypes.byref(op), None)
    assert rc == _native.KM_EINVAL and b"unknown pointwise op" in lib.km_last_error()
    op.kind = _native.OP_GPE_PHASE
    rc = lib.km_mumode(dummy, _native.KM_C128, dummy, _native.KM_C128, dummy, 2, 1, 2, 1,
                       ctypes.byref(op), None)
    assert rc == _native.KM_EINVAL and b"weight" in lib.km_last_error()


def test_tucker_workspace_sizes():
    lib = _native.lib()
    d = 3
    dims = (ctypes.c_int64 * d)(16, 8, 4)
    mats = (ctypes.c_void_p * d)(1, None, 1)
    codes = (ctypes.c_int * d)(_native.KM_C128, 0, _native.KM_F64)
    rows = (ctypes.c_int64 * d)(32, 0, 2)
    nb = ctypes.c_size_t()
    assert lib.km_tucker_workspace(_native.KM_F64, d, dims, mats, codes, rows, ctypes.byref(nb)) == 0
    # largest intermediate: after direction 1 → (32, 8, 4) complex128
    assert nb.value == 32 * 8 * 4 * 16


@pytest.mark.skipif(HAS_CUDA, reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    import paper_2103_01691_b200 as km

    with pytest.raises(km.DeviceError):
        km.mu_mode_product(np.ones((2, 3)), np.eye(3), 2)
    with pytest.raises(km.DeviceError):
        km.step(km.prepare(km.KroneckerOp((np.eye(2),)), 0.1), np.ones(2))


def test_missing_library_fails_loudly(monkeypatch):
    import paper_2103_01691_b200 as km

    monkeypatch.setattr(_native, "_lib", None)
    monkeypatch.setattr(_native, "LIB_PATH", "/nonexistent/libkmb200.so")
    with pytest.raises(km.NativeLibraryError):
        _native.lib()


def test_tucker_buffer_rules_checked_before_launch():
    """ws1 == NULL reuses out as scratch only when the intermediates fit; no aliasing."""
    lib = _native.lib()
    d = 3
    dims = (ctypes.c_int64 * d)(16, 8, 4)
    mats = (ctypes.c_void_p * d)(1, 1, 1)
    codes = (ctypes.c_int * d)(_native.KM_C128, _native.KM_C128, _native.KM_C128)
    rows = (ctypes.c_int64 * d)(32, 8, 2)
    u, out, w0, w1 = (ctypes.c_void_p(a) for a in (0x1000, 0x2000, 0x3000, 0x4000))
    # products 1 and 3 would both write out, but the (32, 8, 4) intermediate is larger than the
    # (32, 8, 2) result: out cannot stand in for ws1
    rc = lib.km_tucker(u, _native.KM_C128, d, dims, mats, codes, rows, out, w0, None, None, None, None)
    assert rc == _native.KM_EINVAL and b"does not fit" in lib.km_last_error()
    for ws0, ws1 in ((u, w1), (w0, u), (w0, out), (w0, w0)):
        rc = lib.km_tucker(u, _native.KM_C128, d, dims, mats, codes, rows, out, ws0, ws1, None, None, None)
        assert rc == _native.KM_EINVAL and b"aliases" in lib.km_last_error()


def test_library_sources_never_allocate_device_memory():
    """kmb200.h promises the library never allocates device memory: every scratch buffer
    (km_tucker's workspaces, the tcgen05 planes, the norm partials, the stream-K scratch)
    is caller-supplied.  No allocation call may appear in the library's sources."""
    csrc = os.path.join(ROOT, "paper_2103_01691_b200", "csrc")
    banned = re.compile(r"\b(cudaMalloc\w*|cuMemAlloc\w*|cudaHostAlloc|cudaMallocHost|cuMemCreate)\s*\(")
    for name in sorted(os.listdir(csrc)):
        if name.endswith((".cu", ".cuh", ".h")):
            text = open(os.path.join(csrc, name)).read()
            assert not banned.search(text), f"{name} allocates device memory"


def test_per_device_state_has_no_process_wide_flags():
    """Set-up the library caches per device (smem opt-ins, cluster occupancy, SM counts) is
    keyed by the device id (memo_get/memo_put, ensure_smem); a process-wide `static bool` or
    `static int` flag would skip the set-up on a second device."""
    csrc = os.path.join(ROOT, "paper_2103_01691_b200", "csrc")
    bad = re.compile(r"static\s+(bool|int)\s+(attr\w*|max_pairs|g_num_sms)\b")
    for name in sorted(os.listdir(csrc)):
        if name.endswith((".cu", ".cuh")):
            assert not bad.search(open(os.path.join(csrc, name)).read()), name


def test_stream_workspace_entry_points():
    lib = _native.lib()
    nb = ctypes.c_size_t()
    if not HAS_CUDA:
        # the size depends on the device's SM count; without a device it still answers
        assert lib.km_stream_workspace_bytes(ctypes.byref(nb)) == 0 and nb.value > 0
    assert lib.km_stream_workspace_bytes(None) == _native.KM_EINVAL
    # too small a workspace is rejected before anything is queued
    rc = lib.km_set_stream_workspace(None, ctypes.c_void_p(0x1000), 16)
    assert rc == _native.KM_EINVAL and b"needed" in lib.km_last_error()
    # unbinding a stream that has no workspace is a no-op
    assert lib.km_set_stream_workspace(None, None, 0) == 0


def test_round2_entry_points_reject_bad_arguments_before_launch():
    lib = _native.lib()
    p = ctypes.c_void_p(0x1000)
    # accumulate must be 0 or 1
    rc = lib.km_mumode_split(p, _native.KM_C128, p, _native.KM_C128, p, 16, 4, 16, 2, 16, 0, 16, 0, 2, None, None)
    assert rc == _native.KM_EINVAL and b"accumulate" in lib.km_last_error()
    # widening pointwise: complex128 -> complex64 would round; widening in place is impossible
    assert lib.km_pointwise_cast(p, _native.KM_C128, ctypes.c_void_p(0x2000), _native.KM_C64, 8, None, None) \
        == _native.KM_EINVAL
    assert lib.km_pointwise_cast(p, _native.KM_C64, p, _native.KM_C128, 8, None, None) == _native.KM_EINVAL
    assert lib.km_pointwise_cast(p, _native.KM_F64, p, _native.KM_F64, 8, None, None) == _native.KM_EINVAL
    # the steps kernel's shape rules: multiples of 32 in [32, 96], steps >= 1
    nb = ctypes.c_size_t()
    for shape, steps in (((48, 64, 64), 1), ((128, 64, 64), 1), ((64, 64, 16), 1), ((64, 64, 64), 0)):
        assert lib.km_steps_small_workspace_bytes(*shape, steps, ctypes.byref(nb)) == _native.KM_EINVAL
    assert lib.km_steps_small_workspace_bytes(64, 64, 64, 10, ctypes.byref(nb)) == 0
    assert nb.value >= 2 * 64**3 * 16 + 30 * 512 * 4
    # a too-small steps workspace, and a misaligned stream-K workspace
    assert lib.km_steps_small(p, p, p, p, 64, 64, 64, 10, p, 16, None) == _native.KM_EINVAL
    big = ctypes.c_size_t()
    assert lib.km_stream_workspace_bytes(ctypes.byref(big)) == 0
    assert lib.km_set_stream_workspace(None, ctypes.c_void_p(0x1008), big.value) == _native.KM_EINVAL


def test_epilogue_norm_contract_checked():
    lib = _native.lib()
    p = ctypes.c_void_p(0x1000)
    op = _native.PointOp()
    op.kind = _native.OP_NONE
    op.d = 3
    op.norm_result = 0x3000  # a result without a partial-sum workspace
    rc = lib.km_mumode(p, _native.KM_C128, p, _native.KM_C128, p, 16, 1, 16, 16, ctypes.byref(op), None)
    assert rc == _native.KM_EINVAL and b"norm" in lib.km_last_error()
    op.norm_ws = 0x4000
    op.norm_ws_count = 4  # too few slots for this product
    rc = lib.km_mumode(p, _native.KM_C128, p, _native.KM_C128, p, 16, 1, 16, 16, ctypes.byref(op), None)
    assert rc == _native.KM_EINVAL and b"slots" in lib.km_last_error()
    # enough for any tiling of m = 256 rows x 65536 fibers
    assert lib.km_norm_epilogue_slots(256, 65536) >= (65536 // 16) * (256 // 16) * 4
