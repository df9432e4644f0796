"""GPU: the promises of include/kmb200.h and of the host mirror around it.

* results handed back to the caller are caller-owned: the page-locked result
  pool never recycles a buffer a numpy view still reads (reference:
  tensor.py:130, 135, 140 return fresh arrays);
* the library never allocates device memory: the stream-K scratch is the
  caller's workspace bound to the stream (km_set_stream_workspace);
* per-device set-up: a second device in the same process gets its own
  shared-memory opt-ins (skipped on a 1-GPU box).
"""

import ctypes

import numpy as np
import pytest

import paper_2103_01691_b200 as km
from oracle import kronmode_oracle as orc

pytestmark = pytest.mark.gpu


def crand(rng, shape):
    return np.asfortranarray(rng.standard_normal(shape) + 1j * rng.standard_normal(shape))


def schrod(n, tau=0.01):
    d2 = km.heat_factors(n, 2).factors[0]
    return km.prepare(km.KroneckerOp((1j * d2,) * 3), tau)


@pytest.mark.parametrize("n", [64, 128])  # 4 MB (to_host pool) and 32 MB (host pipeline)
def test_result_views_survive_later_calls(n):
    rng = np.random.default_rng(n)
    cache = schrod(n)
    u = crand(rng, (n,) * 3)
    r = km.step(cache, u)
    want = orc.step(cache.exps, u)
    plane, real, flat, tr = r[:, :, 0], r.real, r.reshape(-1, order="F"), r.T
    keep = [np.array(x, copy=True) for x in (plane, real, flat, tr)]
    del r  # only views remain
    for _ in range(3):  # same-size calls: a recycled pool buffer would overwrite the views
        km.step(cache, crand(rng, (n,) * 3))
    for view, snap in zip((plane, real, flat, tr), keep):
        assert np.array_equal(view, snap)
    assert orc.rel_l2(plane, want[:, :, 0]) <= 1e-12


def test_pool_buffer_reused_once_all_views_are_gone():
    import gc

    from paper_2103_01691_b200 import _device as dv

    a = dv.pinned_host_array((64, 64, 64), np.complex128)
    addr = a.ctypes.data
    v = a[..., 1]
    del a
    gc.collect()
    b = dv.pinned_host_array((64, 64, 64), np.complex128)
    assert b.ctypes.data != addr  # v still reads the first buffer
    del b, v
    gc.collect()
    c = dv.pinned_host_array((64, 64, 64), np.complex128)
    assert c.ctypes.data == addr  # the first buffer is free again (the second one is too)


def _launch_dir3(lib, u, e, out, n, stream):
    from paper_2103_01691_b200 import _native

    _native.check(lib.km_mumode(u.data_ptr(), _native.KM_C128, e.data_ptr(), _native.KM_C128, out.data_ptr(),
                                n, n * n, n, 1, None, ctypes.c_void_p(stream.cuda_stream)))


def test_streamk_uses_the_bound_workspace_and_never_allocates():
    """160^3 direction-3 product: 4.05 waves of tiles, so the persistent TMA kernel splits its
    last wave (stream-K).  On a fresh stream with a bound workspace the launch must not
    change the device's free memory; on a stream without one it runs whole tiles.  Both
    match the oracle."""
    import torch

    from paper_2103_01691_b200 import _device as dv, _native

    n = 160
    rng = np.random.default_rng(3)
    uh = crand(rng, (n,) * 3)
    eh = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n)
    dev = torch.device("cuda", 0)
    u = dv.to_device(uh, np.complex128, dev)
    e = torch.from_numpy(np.ascontiguousarray(eh)).to(dev)
    want = orc.mu_mode_product(uh, eh, 3)
    lib = _native.lib()
    # warm-up on the default stream (module loading, smem opt-in)
    out0 = torch.empty_like(u)
    _launch_dir3(lib, u, e, out0, n, torch.cuda.current_stream())
    dv.stream_ptr(dev)
    _launch_dir3(lib, u, e, out0, n, torch.cuda.current_stream())
    torch.cuda.synchronize()

    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        dv.stream_ptr(dev)  # binds a torch-allocated workspace to s
        out = torch.empty_like(u)
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info(dev)
    _launch_dir3(lib, u, e, out, n, s)
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info(dev)
    # (the profiler allocates device buffers of its own: look at the kernel name separately)
    from conftest import kernels_launched

    _, names = kernels_launched(lambda: _launch_dir3(lib, u, e, out, n, s))
    # template arguments <KC, op, complex factor, complex tensor, stream-K>
    assert names is None or any("mumode_tma_kernel<false, 0, true, true, true>" in x for x in names), names
    assert free1 >= free0 - (2 << 20), f"the library allocated {(free0 - free1) / 2**20:.1f} MiB"
    assert orc.rel_l2(dv.to_host(dv.as_fortran(out)), want) <= 1e-12

    # unbound stream: whole tiles, same numbers to rounding
    s2 = torch.cuda.Stream(dev)
    out2 = torch.empty_like(u)
    torch.cuda.synchronize()
    _launch_dir3(lib, u, e, out2, n, s2)
    torch.cuda.synchronize()
    assert orc.rel_l2(dv.to_host(dv.as_fortran(out2)), want) <= 1e-12


@pytest.mark.skipif("__import__('torch').cuda.device_count() < 2", reason="needs two GPUs in one process")
def test_second_device_in_the_same_process():
    import torch

    from paper_2103_01691_b200 import _device as dv

    n = 256
    rng = np.random.default_rng(5)
    uh = crand(rng, (n,) * 3)
    eh = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n)
    want = orc.mu_mode_product(uh, eh, 2)
    for idx in (0, 1):
        with torch.cuda.device(idx):
            got = km.mu_mode_product(dv.to_device(uh, np.complex128, torch.device("cuda", idx)), eh, 2)
            assert got.device.index == idx
            assert orc.rel_l2(dv.to_host(got), want) <= 1e-12
