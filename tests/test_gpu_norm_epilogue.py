"""GPU: the epilogue two-norm (km_pointop.norm_result) — the norm of
what the last product stores, from per-warp partial sums in its epilogue, against numpy's
norm of the same output (tensor.py:169-198 "two").  Covers the TMA kernel (whole tiles and
stream-K), the cp.async kernel, real outputs, a fused GPE phase, and the separate-pass
fallback (an op the kernel cannot fuse)."""

import numpy as np
import pytest

import paper_2103_01691_b200 as km
from oracle import kronmode_oracle as orc
from paper_2103_01691_b200 import _device as dv
from paper_2103_01691_b200 import _native

pytestmark = pytest.mark.gpu


def crand(rng, shape):
    return np.asfortranarray(rng.standard_normal(shape) + 1j * rng.standard_normal(shape))


def _norm_op(shape, dev, kind_op=None):
    import torch

    from paper_2103_01691_b200.problems import _attach_norm

    op = kind_op if kind_op is not None else _native.PointOp()
    if kind_op is None:
        op.kind = _native.OP_NONE
        op.d = len(shape)
        for i, n in enumerate(shape):
            op.dims[i] = n
    res = torch.zeros(1, dtype=torch.float64, device=dev)
    keep = []
    _attach_norm(op, res, dev, keep)
    return op, res, keep


@pytest.mark.parametrize("shape,real", [((256, 256, 256), False), ((64, 64, 64), False), ((160, 160, 160), False),
                                        ((96, 80, 72), False), ((128, 128, 64), True)])
def test_epilogue_norm_of_a_step(shape, real):
    import torch

    from paper_2103_01691_b200.tensor import run_tucker

    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(sum(shape))
    u = np.asfortranarray(rng.standard_normal(shape)) if real else crand(rng, shape)
    mats = [(rng.standard_normal((n, n)) if real else rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
            / np.sqrt(n) for n in shape]
    t = dv.to_device(u, u.dtype, dev)
    op, res, keep = _norm_op(shape, dev)
    out = run_tucker(t, mats, post=op, keepalive=keep)
    host = dv.to_host(out)
    want = np.linalg.norm(host.ravel())
    assert float(res.item()) == pytest.approx(want, rel=1e-13)
    assert orc.rel_l2(host, orc.tucker(u, mats)) <= 1e-12


def test_epilogue_norm_with_fused_gpe_phase_and_run():
    import torch

    from paper_2103_01691_b200.problems import weighted_vortex_state

    dev = torch.device("cuda", 0)
    n = 128
    grids, lin_op, weights = km.gpe_setup(n)
    psi = weighted_vortex_state(grids, weights)
    cache = km.prepare(lin_op, 0.1)
    t = dv.to_device(psi, np.complex128, dev)
    res = torch.zeros(1, dtype=torch.float64, device=dev)
    out = km.gpe_strang_run(cache, weights, t, 0.1, 3, _norm_out=res)
    host = dv.to_host(out)
    assert float(res.item()) == pytest.approx(np.linalg.norm(host.ravel()), rel=1e-13)
    plain = dv.to_host(km.gpe_strang_run(cache, weights, t, 0.1, 3))
    assert np.array_equal(host, plain)  # asking for the norm does not change the state


def test_epilogue_norm_fallback_pass():
    """A diagonal phase along direction 1 is not fusable into the direction-3 epilogue: the
    product, the phase pass, then the norm as a separate pass — same contract."""
    import torch

    from paper_2103_01691_b200.problems import _diag_op
    from paper_2103_01691_b200.tensor import run_tucker

    dev = torch.device("cuda", 0)
    shape = (48, 40, 36)
    rng = np.random.default_rng(7)
    u = crand(rng, shape)
    mats = [None, None, (rng.standard_normal((36, 36)) + 1j * rng.standard_normal((36, 36))) / 6]
    f = np.exp(1j * rng.standard_normal(48))
    f_d = dv.cached_vector(f, np.complex128, dev)
    op = _diag_op(shape, f_d, 0)
    op, res, keep = _norm_op(shape, dev, op)
    out = dv.to_host(run_tucker(dv.to_device(u, np.complex128, dev), mats, post=op, keepalive=keep + [f_d]))
    want = orc.mu_mode_product(u, mats[2], 3) * f.reshape(48, 1, 1)
    assert orc.rel_l2(out, want) <= 1e-12
    assert float(res.item()) == pytest.approx(np.linalg.norm(out.ravel()), rel=1e-13)


def test_gpe_driver_drift_uses_the_epilogue_norm():
    from paper_2103_01691_b200.drivers import gpe_run

    rep = gpe_run(32, T=0.3, tau=0.1)
    assert 0.0 <= rep.error < 1e-10  # the Strang flow conserves the weighted two-norm
