"""CPU, world size 2 (gloo): the multi-GPU slab decomposition's schedule and
block layouts (paper_2103_01691_b200/dist.py) against the single-process
oracle.  The products run through the oracle with the kernel's blocked
(split) addressing emulated in numpy; the exchange is a real
torch.distributed all_to_all_single over gloo.  The GPU kernels' split
addressing itself is covered by the virtual-rank test in test_gpu_dist.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

from oracle import kronmode_oracle as orc
from paper_2103_01691_b200 import dist


def gather_in(buf, nl, nmu, nr, kcb, kbs):
    if kcb == nmu:
        return buf[: nl * nmu * nr].reshape((nl, nmu, nr), order="F")
    blocks = [buf[b * kbs: b * kbs + nl * kcb * nr].reshape((nl, kcb, nr), order="F") for b in range(nmu // kcb)]
    return np.concatenate(blocks, axis=1)


def scatter_out(buf, x, ncb, nbs):
    nl, m, nr = x.shape
    if ncb == m:
        buf[: x.size] = x.reshape(-1, order="F")
        return
    for b in range(m // ncb):
        buf[b * nbs: b * nbs + nl * ncb * nr] = x[:, b * ncb:(b + 1) * ncb, :].reshape(-1, order="F")


class CpuSlabStepper(dist.SlabStepper):
    """SlabStepper whose products run on the CPU oracle (test double for the kernels): the
    schedule (serial or two-half overlapped), the blocked addressing and the derived forms of
    E3 are the stepper's own; only the product itself is the oracle's."""

    def __init__(self, plan, rank, local_a, mats_np, comm, overlap=True):
        self.plan, self.rank, self.comm = plan, rank, comm
        self.mats = list(mats_np)
        self.a = local_a.copy()
        self.w = np.empty_like(self.a)
        self.send = torch.zeros(self.a.size, dtype=torch.complex128)
        self.recv = torch.zeros(self.a.size, dtype=torch.complex128)
        self.layout = "A"
        self.overlap = overlap and plan.overlap_ok()
        self.derived = {}
        if self.overlap:
            self._derive(self.mats[2])
        self._works = []

    def _derive(self, e3):
        for h, pi in enumerate(self.plan.e3_column_halves()):
            self.derived[f"E3p{h}"] = e3[:, pi]
        for g, rho in enumerate(self.plan.e3_row_halves()):
            self.derived[f"E3r{g}"] = e3[rho, :]

    def _np(self, key):
        b = self._buf(key)
        return b.numpy() if isinstance(b, torch.Tensor) else b

    def _exec(self, prods, post=None):
        for p in prods:
            src = self._np(p.src)[p.soff:]
            dst = self._np(p.dst)[p.doff:]
            x = gather_in(src, p.nl, p.nmu, p.nr, p.kcb, p.kbs)
            y = orc.mu_mode_product(x, self._mat(p.mat), 2)
            if p.acc:
                y = gather_in(dst, p.nl, p.m, p.nr, p.m, 0) + y
            scatter_out(dst, y, p.ncb, p.nbs)
        if post is not None:
            self._phase(self.a, post)


class CpuGpeStepper(CpuSlabStepper, dist.SlabGpeStepper):
    """SlabGpeStepper's schedule with the phases as numpy (oracle nonlinear_half on the local
    slab's weights, cut from the global vectors exactly as the device ops' pointer offsets)."""

    def __init__(self, plan, rank, local_a, mats_np, comm, weights, half_tau, overlap=True):
        CpuSlabStepper.__init__(self, plan, rank, local_a, mats_np, comm, overlap)
        self.weights = [np.asarray(w, dtype=float) for w in weights]
        self.half_tau = half_tau

    def _op(self, layout, repeat):
        return (layout, repeat)

    def _phase(self, buf, op):
        layout, repeat = op
        n1, n2, n3 = self.plan.dims
        c2, c3, r = self.plan.c2, self.plan.c3, self.rank
        w1, w2, w3 = self.weights
        if layout == "A":
            shape, ws = (n1, n2, c3), (w1, w2, w3[r * c3:(r + 1) * c3])
        else:
            shape, ws = (n1, c2, n3), (w1, w2[r * c2:(r + 1) * c2], w3)
        b = buf.numpy() if isinstance(buf, torch.Tensor) else buf
        x = b.reshape(shape, order="F")
        wp = orc.weight_product(ws, shape)
        for _ in range(repeat):
            x = orc.nonlinear_half(x, wp, self.half_tau)
        b[:] = x.reshape(-1, order="F")


class CpuTdpotStepper(CpuSlabStepper, dist.SlabTdpotStepper):
    """SlabTdpotStepper's schedule with the per-step fold of E3 in numpy."""

    def __init__(self, plan, rank, local_a, mats_np, comm, x_nodes, overlap=True):
        CpuSlabStepper.__init__(self, plan, rank, local_a, list(mats_np), comm, overlap)
        self.e3 = mats_np[2]
        self.xn = np.asarray(x_nodes, dtype=float)

    def begin_step(self, t=0.0, tau=0.0, **kw):
        c_a, c_b = orc.sin2_integral(t, t + 0.5 * tau), orc.sin2_integral(t + 0.5 * tau, t + tau)
        self.mats[2] = (np.exp(-1j * self.xn * c_b)[:, None] * self.e3) * np.exp(-1j * self.xn * c_a)[None, :]
        if self.overlap:
            self._derive(self.mats[2])
        return dist.SlabStepper.begin_step(self)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, dims, steps, q, overlap=True):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(3)
        u = np.asfortranarray(rng.standard_normal(dims) + 1j * rng.standard_normal(dims))
        mats = [rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)) for n in dims]
        mats = [m / np.linalg.norm(m, 2) for m in mats]
        plan = dist.SlabPlan(dims, world)
        local = np.asfortranarray(plan.slab_a(u, rank)).reshape(-1, order="F")
        st = CpuSlabStepper(plan, rank, local, mats, dist.NcclExchange(), overlap)
        for _ in range(steps):
            st.step()
        want = u
        for _ in range(steps):
            want = orc.step(mats, want)
        shape = plan.shape_a if st.layout == "A" else plan.shape_b
        got = st.a.reshape(shape, order="F")
        ref = plan.slab_a(want, rank) if st.layout == "A" else plan.slab_b(want, rank)
        q.put((rank, st.layout, orc.rel_l2(got, ref)))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("overlap", [False, True])
@pytest.mark.parametrize("steps", [1, 2, 3])
def test_slab_schedule_world2_matches_oracle(steps, overlap):
    """Serial schedule and the two-half overlapped one (asynchronous all-to-all per half,
    permuted E3 columns on even steps, E3 row halves on odd steps)."""
    world, dims = 2, (6, 32, 64)
    assert dist.SlabPlan(dims, world).overlap_ok()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, steps, q, overlap)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    for rank, layout, err in res:
        assert layout == ("B" if steps % 2 else "A")
        assert err <= 1e-13, (rank, err)


def test_slab_plan_rejects_uneven_split():
    with pytest.raises(ValueError):
        dist.SlabPlan((8, 10, 8), 4)


def test_slab_plan_blocks_partition_the_slab():
    plan = dist.SlabPlan((4, 8, 8), 4)
    assert plan.block * plan.P == plan.local
    assert plan.shape_a == (4, 8, 2) and plan.shape_b == (4, 2, 8)


def _splitting_worker(rank, world, port, dims, steps, kind, q, overlap=True):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(7)
        u = np.asfortranarray(rng.standard_normal(dims) + 1j * rng.standard_normal(dims)) * 0.7
        mats = [rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)) for n in dims]
        mats = [m / np.linalg.norm(m, 2) for m in mats]
        plan = dist.SlabPlan(dims, world)
        local = np.asfortranarray(plan.slab_a(u, rank)).reshape(-1, order="F")
        tau = 0.1
        if kind == "gpe":
            ws = [rng.random(n) + 0.5 for n in dims]
            st = CpuGpeStepper(plan, rank, local, mats, dist.NcclExchange(), ws, 0.5 * tau, overlap)
            st.run(steps)
            want = u
            for _ in range(steps):
                want = orc.gpe_strang_step(mats, ws, want, tau)
        else:
            x = np.linspace(-3.0, 3.0, dims[2])
            st = CpuTdpotStepper(plan, rank, local, mats, dist.NcclExchange(), x, overlap)
            st.run(0.25, tau, steps)
            want = u
            for s_ in range(steps):
                want = orc.tdpot_strang_step(mats, x, want, 0.25 + s_ * tau, tau)
        shape = plan.shape_a if st.layout == "A" else plan.shape_b
        got = st.a.reshape(shape, order="F")
        ref = plan.slab_a(want, rank) if st.layout == "A" else plan.slab_b(want, rank)
        q.put((rank, st.layout, orc.rel_l2(got, ref)))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("overlap", [False, True])
@pytest.mark.parametrize("kind", ["gpe", "tdpot"])
@pytest.mark.parametrize("steps", [1, 2])
def test_sharded_splitting_world2_matches_oracle(kind, steps, overlap):
    """Configs 4 and 5 sharded: GPE Strang steps (phases on slab-offset weights, closing and
    opening half-phases merged between steps) and TD-potential Strang steps (E3 folded per
    step) over world-size 2 gloo, against the single-process oracle."""
    world, dims = 2, (6, 32, 64)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_splitting_worker, args=(r, world, port, dims, steps, kind, q, overlap))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    for rank, layout, err in res:
        assert layout == ("B" if steps % 2 else "A")
        assert err <= 1e-13, (rank, err)
