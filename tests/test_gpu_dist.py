"""GPU: the slab decomposition's kernels (blocked input/output addressing of
km_mumode_split) and the virtual-rank schedule on one device, against the
single-GPU stepper and the oracle."""

import ctypes

import numpy as np
import pytest

import paper_2103_01691_b200 as km
from oracle import kronmode_oracle as orc
from paper_2103_01691_b200 import _device as dv
from paper_2103_01691_b200 import _native, dist

pytestmark = pytest.mark.gpu


def crand(rng, shape):
    return np.asfortranarray(rng.standard_normal(shape) + 1j * rng.standard_normal(shape))


def test_split_kernel_addressing():
    import torch

    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(5)
    nl, nmu, nr, m = 24, 64, 5, 48
    kcb, ncb = 16, 8
    x = crand(rng, (nl, nmu, nr))
    L = rng.standard_normal((m, nmu)) + 1j * rng.standard_normal((m, nmu))
    want = orc.mu_mode_product(x, L, 2)
    kbs = nl * kcb * nr + 7  # padded block stride: the stride is honoured, not assumed
    nbs = nl * ncb * nr + 3
    src = np.zeros((nmu // kcb) * kbs, dtype=np.complex128)
    for b in range(nmu // kcb):
        src[b * kbs: b * kbs + nl * kcb * nr] = x[:, b * kcb:(b + 1) * kcb, :].reshape(-1, order="F")
    src_d = torch.from_numpy(src).to(dev)
    out_d = torch.zeros((m // ncb) * nbs, dtype=torch.complex128, device=dev)
    L_d = torch.from_numpy(np.ascontiguousarray(L)).to(dev)
    _native.check(_native.lib().km_mumode_split(
        src_d.data_ptr(), _native.KM_C128, L_d.data_ptr(), _native.KM_C128, out_d.data_ptr(),
        m, nl, nmu, nr, kcb, kbs, ncb, nbs, 0, None, dv.stream_ptr(dev)))
    out = out_d.cpu().numpy()
    got = np.concatenate([out[b * nbs: b * nbs + nl * ncb * nr].reshape((nl, ncb, nr), order="F")
                          for b in range(m // ncb)], axis=1)
    assert orc.rel_l2(got, want) <= 1e-14


def test_split_rejects_bad_blocks():
    lib = _native.lib()
    p = ctypes.c_void_p(16)
    assert lib.km_mumode_split(p, 3, p, 3, p, 16, 4, 20, 2, 10, 40, 16, 0, 0, None, None) == _native.KM_EINVAL
    assert lib.km_mumode_split(p, 3, p, 3, p, 16, 1, 32, 2, 16, 64, 16, 0, 0, None, None) == _native.KM_EINVAL


@pytest.mark.parametrize("P,n,steps,exchange,overlap", [
    (2, 64, 3, "nccl", True), (4, 64, 4, "nccl", True), (8, 256, 3, "nccl", True), (8, 256, 2, "nccl", False),
    (4, 256, 2, "nccl", True), (2, 64, 3, "peer", False), (4, 64, 4, "peer", False), (8, 256, 3, "peer", False),
    (2, 256, 2, "peer", False)])
def test_virtual_ranks_match_single_gpu(P, n, steps, exchange, overlap):
    import torch

    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(0)
    u = crand(rng, (n,) * 3)
    d2 = km.heat_factors(n, 2).factors[0]
    cache = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
    grp = dist.VirtualSlabGroup(u, cache, dev, P, exchange=exchange, overlap=overlap)
    if exchange == "nccl":
        assert grp.ranks[0].overlap == (overlap and grp.plan.overlap_ok())
    for _ in range(steps):
        grp.step()
    got = grp.gather()
    ref = dist.LocalStepper(dv.to_device(u, np.complex128, dev), cache.device_exps((np.complex128,) * 3, dev))
    for _ in range(steps):
        ref.step()
    want = dv.to_host(ref.state)
    assert orc.rel_l2(got, want) <= 1e-12
    if n <= 64:
        o = u
        for _ in range(steps):
            o = orc.step(cache.exps, o)
        assert orc.rel_l2(got, o) <= 1e-12


@pytest.mark.parametrize("P,n,steps,overlap", [(2, 64, 3, True), (4, 64, 2, True), (8, 128, 3, True),
                                               (8, 256, 2, True), (8, 256, 3, False)])
def test_virtual_ranks_gpe_strang(P, n, steps, overlap):
    """Config 5 sharded: GPE Strang steps on P virtual slab ranks against the oracle's step
    loop (problems.py:548-565, 597-598) and the single-GPU fused run."""
    import torch

    from paper_2103_01691_b200.problems import weighted_vortex_state

    dev = torch.device("cuda", 0)
    grids, lin_op, weights = km.gpe_setup(n)
    psi = weighted_vortex_state(grids, weights)
    tau = 0.1
    cache = km.prepare(lin_op, tau)
    grp = dist.VirtualSlabGroup(psi, cache, dev, P, kind="gpe", weights=weights, tau=tau, overlap=overlap)
    for k in range(steps):
        grp.step(k=k, steps=steps)
    got = grp.gather()
    want = psi
    for _ in range(steps):
        want = orc.gpe_strang_step(cache.exps, weights, want, tau)
    assert orc.rel_l2(got, want) <= 1e-12
    single = km.gpe_strang_run(cache, weights, psi, tau, steps)
    assert orc.rel_l2(got, single) <= 1e-13


@pytest.mark.parametrize("P,n,steps,overlap", [(2, 32, 3, True), (2, 64, 3, True), (4, 64, 2, True),
                                               (8, 256, 3, True), (8, 256, 2, False)])
def test_virtual_ranks_tdpot_strang(P, n, steps, overlap):
    """Config 4 sharded (256^3 over 8 ranks): E3 folded per step on every rank."""
    import torch

    from paper_2103_01691_b200.hermite import physical_propagator
    from paper_2103_01691_b200.problems import schrodinger_initial_state

    dev = torch.device("cuda", 0)
    b = km.hermite_basis(n)
    tau = 0.02
    p = physical_propagator(b, tau)
    cache = km.PropagatorCache(tau, (p, p, p))
    psi = schrodinger_initial_state((b.nodes,) * 3)
    grp = dist.VirtualSlabGroup(psi, cache, dev, P, kind="tdpot", x_nodes=b.nodes, overlap=overlap)
    for s_ in range(steps):
        grp.step(t=s_ * tau, tau=tau)
    got = grp.gather()
    want = psi
    for s_ in range(steps):
        want = orc.tdpot_strang_step(cache.exps, b.nodes, want, s_ * tau, tau)
    assert orc.rel_l2(got, want) <= 1e-12
